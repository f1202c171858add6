mkdir -p gpurun_out/s4k
timeout 900 python -m pytest tests/test_gpu_ods.py -q -x -k "one_context_per_shard or across_processes" > gpurun_out/s4k/t.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/s4k/t.log
