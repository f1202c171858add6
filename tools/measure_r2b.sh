#!/bin/bash
# Round-2 final measurement pass (run under gpurun from the repo root).  The ncu
# reports are summarised on the box and deleted (gpurun copies back <= 64 MiB).
TAG=${1:-r2b}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv > $OUT/gpu.txt
python tools/wbw.py > $OUT/write_bandwidth.txt 2>&1
timeout 1500 python -m pytest tests -q -m gpu > $OUT/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -1 $OUT/gpu_tests.log
timeout 300 python __graft_entry__.py smoke > $OUT/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $OUT/smoke.log
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"
timeout 900 python bench.py > $OUT/bench_repeat.json 2>> $OUT/bench.err; echo "bench2 rc=$?"
timeout 600 python bench.py --workload imagenet1k --evict-tiers 1 --replicas 0 --extra-workloads "" --shards "" --no-cpu-baseline > $OUT/bench_imagenet1k_evictall.json 2>> $OUT/bench.err; echo "evictall rc=$?"
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $OUT/bench_reference.json 2>> $OUT/bench.err; echo "reference rc=$?"
SENECA_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 2 --warmup 3 --no-shard-replay \
  --mdp-large 0 > $OUT/bench_gloo2.json 2> $OUT/bench_gloo2.err; echo "gloo2 rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
  python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-profile --replicas 0 --shards "" --mdp-large 0 \
  > /dev/null 2>&1; echo "ncu launches rc=$?"
ARGS=""
for w in imagenet22k imagenet1k openimages; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:ods_rounds -c 1 -o $OUT/ncu_ods_rounds_$w \
    python tools/profile_ods.py $w 1000000 --plain > /dev/null 2>&1; echo "ncu ods $w rc=$?"
  ARGS="$ARGS ods_rounds@$w=$OUT/ncu_ods_rounds_$w.ncu-rep"
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:mdp_sweep -s 1 -c 1 -o $OUT/ncu_mdp_sweep \
  python tools/profile_mdp.py 10000 > /dev/null 2>&1; echo "ncu mdp rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:mdp_sweep -s 1 -c 1 -o $OUT/ncu_mdp_sweep_100k \
  python tools/profile_mdp.py 100000 > /dev/null 2>&1; echo "ncu mdp100k rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ods_recount_all -c 1 -o $OUT/ncu_recount_imagenet22k \
  python tools/profile_ods.py imagenet22k 1 > /dev/null 2>&1; echo "ncu recount rc=$?"
ARGS="$ARGS mdp_sweep@10000x5151=$OUT/ncu_mdp_sweep.ncu-rep mdp_sweep@100000x5151=$OUT/ncu_mdp_sweep_100k.ncu-rep ods_recount_all@imagenet22k=$OUT/ncu_recount_imagenet22k.ncu-rep"
python tools/ncu_summary.py $OUT/ncu_summary.md $OUT/ncu_traffic.json $ARGS > $OUT/ncu_summary.log 2>&1; echo "summary rc=$?"
python tools/ncu_lines.py $OUT/ncu_ods_rounds_imagenet22k.ncu-rep 40 > $OUT/ncu_lines_imagenet22k.txt 2>&1
python tools/ncu_lines.py $OUT/ncu_mdp_sweep.ncu-rep 40 --by-inst > $OUT/ncu_lines_mdp_by_inst.txt 2>&1
ls -la $OUT/*.ncu-rep > $OUT/ncu_reports.txt 2>&1
rm -f $OUT/*.ncu-rep
