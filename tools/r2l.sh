#!/bin/bash
T=${1:-r2l}; mkdir -p gpurun_out/$T
timeout 600 python -m pytest tests/test_gpu_mdp.py -q -x > gpurun_out/$T/tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/$T/tests.log
V="variants/m_base.so variants/m_gtab.so"
timeout 300 python tools/mdp_variants.py $V 2>&1 | tee gpurun_out/$T/mdp10k.txt
MDP_N=100000 timeout 300 python tools/mdp_variants.py $V 2>&1 | tee gpurun_out/$T/mdp100k.txt
timeout 600 python bench.py --workload imagenet1k --replicas 0 --shards "" --mdp-large 0 --no-cpu-baseline --extra-workloads "" > gpurun_out/$T/bench_in1k.json 2> gpurun_out/$T/bench_in1k.err; echo "bench rc=$?"
python -c "import json;d=json.loads(open('gpurun_out/$T/bench_in1k.json').read().strip().splitlines()[-1]);print(d['value']/1e6, d['mdp']['ms_per_step'], d['mdp']['roofline']['frac']);print(json.dumps(d['ods_round_phase_share']))"
