# A/B of the clustered round launch (SENECA_ROUND_CLUSTER) on ImageNet-1K, interleaved
mkdir -p gpurun_out/s4q
for i in 1 2 3 4 5; do
  for cl in 0 1; do
    SENECA_ROUND_CLUSTER=$cl timeout 300 python bench.py --workload imagenet1k --no-cpu-baseline --replicas 0 --steps 2 --warmup 1 --extra-workloads "" --mdp-large 0 --shards "" > gpurun_out/s4q/cl${cl}_$i.json 2> gpurun_out/s4q/cl${cl}_$i.err
    python -c "import json;d=json.loads(open('gpurun_out/s4q/cl${cl}_$i.json').read().strip().splitlines()[-1]);print('cluster=$cl $i', round(d['value']/1e6,1), round(d['ms_per_step']*1e3/d['config']['rounds_per_step'],3), d['parity']['ods_vs_oracle_golden'])" 2>/dev/null || (echo "cluster=$cl $i FAILED"; tail -3 gpurun_out/s4q/cl${cl}_$i.err)
  done
done
SENECA_ROUND_CLUSTER=1 timeout 600 python -m pytest tests/test_gpu_ods.py -q -x -k "toy or imagenet1k or cold or arriv" > gpurun_out/s4q/t.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/s4q/t.log
