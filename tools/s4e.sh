bash tools/odsab.sh s4e imagenet1k 3 base fast2 fast3
timeout 900 python -m pytest tests/test_gpu_ods.py -q -x > gpurun_out/s4e/ods_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/s4e/ods_tests.log
timeout 300 python bench.py --workload imagenet1k --no-cpu-baseline --replicas 0 --steps 2 --warmup 3 --extra-workloads "" --mdp-large 0 --shards "" > gpurun_out/s4e/in1k.json 2> gpurun_out/s4e/in1k.err; echo rc=$?
