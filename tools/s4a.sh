OUT=gpurun_out/s4a; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/gpu.txt
timeout 1500 python -m pytest tests -q -m gpu -x > $OUT/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -3 $OUT/gpu_tests.log
timeout 300 python __graft_entry__.py smoke > $OUT/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"; tail -3 $OUT/bench.err
