mkdir -p gpurun_out/s4h
timeout 900 python -m pytest tests/test_gpu_ods.py -q -x -k "sharded or storage_list or late" > gpurun_out/s4h/t.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/s4h/t.log
timeout 600 python bench.py --no-cpu-baseline --replicas 0 --steps 2 --warmup 3 --extra-workloads "" --mdp-large 0 --shards 2,4,8 > gpurun_out/s4h/b.json 2> gpurun_out/s4h/b.err; echo rc=$?
python -c "import json;d=json.loads(open('gpurun_out/s4h/b.json').read().strip().splitlines()[-1]);print(d['value']/1e6, d['config']['us_per_round']);[print(x['shards'], round(x['us_per_round'],2), round(x['value']/1e6,1), x['parity']) for x in d['sharded']['runs']]"
