OUT=gpurun_out/s4b; mkdir -p $OUT
timeout 600 python bench.py --workload imagenet1k --no-cpu-baseline --replicas 0 --steps 2 --warmup 3 --extra-workloads "" --mdp-large 0 --shards "" > $OUT/in1k.json 2> $OUT/in1k.err; echo rc=$?
