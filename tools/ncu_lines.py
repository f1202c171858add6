"""Top source lines (--by-inst: by instructions executed) of an ncu report by warp-stall samples (needs -lineinfo and
--import-source on):  python tools/ncu_lines.py REPORT [N] [--nobar]
--nobar ranks lines by samples that are not barrier waits (where the slowest
warps spend their time between barriers)."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2].isdigit() else 40
nobar = "--nobar" in sys.argv
byinst = "--by-inst" in sys.argv     # rank by warp instructions executed instead
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
agg, reasons = {}, {}
fname = hdr = None
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 8 or r[0] == "":
        continue
    try:
        line = int(r[0])
        samp = int(r[4])
        ins = int(r[7])
    except ValueError:
        continue
    st = {}
    for k, name in enumerate(hdr):
        if name.startswith("stall_") and "Not Issued" not in name:
            try:
                st[name[6:]] = int(r[k])
            except ValueError:
                pass
    for k, v in st.items():
        reasons[k] = reasons.get(k, 0) + v
    key = samp - st.get("barrier", 0) if nobar else samp
    top3 = ",".join(f"{k}:{v}" for k, v in sorted(st.items(), key=lambda kv: -kv[1])[:3] if v)
    agg[(fname, line)] = (key, ins, r[1].strip()[:80], top3)
tot = sum(v[0] for v in agg.values())
print(f"total samples {tot}; by reason:",
      ", ".join(f"{k} {100*v/max(1,sum(reasons.values())):.1f}%" for k, v in sorted(reasons.items(), key=lambda kv: -kv[1])[:9]))
for (f, l), (s, i, src, t3) in sorted(agg.items(), key=lambda kv: -kv[1][1 if byinst else 0])[:top]:
    print(f"{100*s/tot:5.1f}% inst{i:10d} {f}:{l:<5d} {src:80s} {t3}")
