# DSMEM signals (cluster launch) vs global signals (cluster launch), ImageNet-1K, interleaved; then the coupled GPU tests
mkdir -p gpurun_out/s4s
SENECA_DSMEM_SIGNALS=1 timeout 120 python tools/profile_ods.py toy 96 --plain > gpurun_out/s4s/toy.log 2>&1; echo "toy rc=$?"
for i in 1 2 3 4; do
  for ds in 0 1; do
    SENECA_DSMEM_SIGNALS=$ds timeout 300 python bench.py --workload imagenet1k --no-cpu-baseline --replicas 0 --steps 2 --warmup 1 --extra-workloads "" --mdp-large 0 --shards "" > gpurun_out/s4s/ds${ds}_$i.json 2> gpurun_out/s4s/ds${ds}_$i.err
    python -c "import json;d=json.loads(open('gpurun_out/s4s/ds${ds}_$i.json').read().strip().splitlines()[-1]);print('dsmem=$ds $i', round(d['value']/1e6,1), round(d['ms_per_step']*1e3/d['config']['rounds_per_step'],3), d['parity']['ods_vs_oracle_golden'])" 2>/dev/null || (echo "dsmem=$ds $i FAILED"; tail -3 gpurun_out/s4s/ds${ds}_$i.err)
  done
done
timeout 900 python -m pytest tests/test_gpu_ods.py -q -x > gpurun_out/s4s/t.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/s4s/t.log
