T=${1:-mdp3}; mkdir -p gpurun_out/$T
timeout 300 python -m pytest tests/test_gpu_mdp.py -q -x > gpurun_out/$T/t.log 2>&1; echo rc=$?; tail -1 gpurun_out/$T/t.log
timeout 300 python bench.py --workload toy --no-cpu-baseline > gpurun_out/$T/bench_toy.json 2>gpurun_out/$T/b.err; echo brc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:mdp_sweep -c 1 -o gpurun_out/$T/ncu_mdp python tools/profile_ods.py toy 10 --mdp > /dev/null 2>&1; echo nrc=$?
