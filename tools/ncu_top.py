"""Print the headline metrics of an ncu report (first kernel): time, DRAM
traffic, throughput, occupancy, issue, the busiest pipes and the top stalls."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h, v = rows[0], rows[2]
val = {}
for k, x in zip(h, v):
    try:
        val[k] = float(x.replace(",", ""))
    except ValueError:
        pass
for k in ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
          "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
          "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__inst_executed.sum",
          "launch__registers_per_thread", "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem"]:
    if k in val:
        print(f"{k:70s} {val[k]:.4g}")
pipes = sorted(((x, k) for k, x in val.items() if k.startswith("sm__inst_executed_pipe_") and
                k.endswith(".avg.pct_of_peak_sustained_active")), reverse=True)[:6]
for x, k in pipes:
    print(f"{k:70s} {x:.1f}")
for k in ["l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
          "SM_A.TriageCompute.sm__inst_executed_pipe_xu_realtime.avg.pct_of_peak_sustained_elapsed"]:
    if k in val:
        print(f"{k:70s} {val[k]:.1f}")
st = sorted(((x, k) for k, x in val.items() if k.startswith("smsp__average_warp_latency_issue_stalled_") and
             k.endswith(".ratio")), reverse=True)[:6]
for x, k in st:
    print(f"{k:70s} {x:.2f}")
