OUT=gpurun_out/final; mkdir -p $OUT
timeout 1500 python -m pytest tests -q -m gpu > $OUT/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -1 $OUT/gpu_tests.log
timeout 300 python __graft_entry__.py smoke > $OUT/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $OUT/smoke.log
