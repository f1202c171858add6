#!/bin/bash
# Full measurement pass on a GPU box (run under gpurun from the repo root):
#   tests, smoke, bench (all ODS workloads), reference arm, ncu launch list and
#   full captures of the two kernels.  Artifacts land in gpurun_out/$TAG/.
TAG=${1:-r1}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv > $OUT/gpu.txt
timeout 900 python -m pytest tests -q -m gpu > $OUT/gpu_tests.log 2>&1; echo "gpu tests rc=$?"; tail -1 $OUT/gpu_tests.log
timeout 300 python __graft_entry__.py smoke > $OUT/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $OUT/smoke.log
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"
for w in openimages imagenet22k; do
  timeout 600 python bench.py --workload $w --no-cpu-baseline > $OUT/bench_$w.json 2>> $OUT/bench.err; echo "bench $w rc=$?"
done
for w in imagenet1k imagenet22k; do   # the second eviction mode (R-O21), gated by its oracle golden
  timeout 600 python bench.py --workload $w --evict-tiers 1 --replicas 0 --no-cpu-baseline > $OUT/bench_${w}_evictall.json 2>> $OUT/bench.err; echo "bench $w evict-all rc=$?"
done
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $OUT/bench_reference.json 2>> $OUT/bench.err; echo "reference rc=$?"
# launch list of one bench step (cold, serialised: compare shares, not absolutes)
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
  python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-profile > /dev/null 2>&1; echo "ncu launches rc=$?"
# full captures of the launches bench.py times: each workload's whole replay
# (one ods_rounds launch) and the 10,000-profile MDP sweep with the grid
for w in imagenet1k openimages imagenet22k; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:ods_rounds -c 1 -o $OUT/ncu_ods_rounds_$w \
    python tools/profile_ods.py $w 1000000 --plain > /dev/null 2>&1; echo "ncu ods $w rc=$?"
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:mdp_sweep -c 1 -o $OUT/ncu_mdp_sweep \
  python tools/profile_ods.py toy 10 --mdp > /dev/null 2>&1; echo "ncu mdp rc=$?"
# the init bitmap pass (ods_recount_all) at ImageNet-22K size
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ods_recount_all -c 1 -o $OUT/ncu_recount_imagenet22k \
  python tools/profile_ods.py imagenet22k 1 > /dev/null 2>&1; echo "ncu recount rc=$?"
