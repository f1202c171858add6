OUT=gpurun_out/s4c; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_ods.py -q -x > $OUT/ods_tests.log 2>&1; echo "tests rc=$?"; tail -2 $OUT/ods_tests.log
bash tools/odsab.sh s4c imagenet1k 3 base fast
timeout 300 python bench.py --workload imagenet1k --no-cpu-baseline --replicas 0 --steps 2 --warmup 3 --extra-workloads "" --mdp-large 0 --shards "" > $OUT/in1k.json 2> $OUT/in1k.err; echo rc=$?
