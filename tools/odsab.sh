# bash tools/odsab.sh TAG WORKLOAD REPEATS lib1 lib2 ...: interleaved repeats of one workload per variant
TAG=$1; W=$2; N=$3; shift 3
mkdir -p gpurun_out/$TAG
for i in $(seq 1 $N); do
  for v in "$@"; do
    SENECA_LIB=$PWD/variants/$v.so timeout 300 python bench.py --workload $W --no-cpu-baseline --replicas 0 --steps 2 --warmup 1 --extra-workloads "" --mdp-large 0 --shards "" > gpurun_out/$TAG/${v}_${W}_$i.json 2> /dev/null
    python -c "import json;d=json.loads(open('gpurun_out/$TAG/${v}_${W}_$i.json').read().strip().splitlines()[-1]);print('$v $W $i', round(d['value']/1e6,1), round(d['ms_per_step']*1e3/d['config']['rounds_per_step'],3), d['parity']['ods_vs_oracle_golden'])" 2>/dev/null || echo "$v $W $i FAILED"
  done
done
