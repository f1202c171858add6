# bash tools/odsvar.sh TAG lib1 lib2 ...: bench each ODS library variant on the three workloads
TAG=$1; shift
mkdir -p gpurun_out/$TAG
for v in "$@"; do
  for w in imagenet1k imagenet22k openimages; do
    SENECA_LIB=$PWD/variants/$v.so timeout 300 python bench.py --workload $w --no-cpu-baseline --replicas 0 --steps 2 --warmup 1 --extra-workloads "" --mdp-large 0 > gpurun_out/$TAG/${v}_$w.json 2> gpurun_out/$TAG/${v}_$w.err
    python -c "import json;d=json.loads(open('gpurun_out/$TAG/${v}_$w.json').read().strip().splitlines()[-1]);print('$v $w', round(d['value']/1e6,1), round(d['ms_per_step']*1e3/d['config']['rounds_per_step'],2), d['parity']['ods_vs_oracle_golden'])" 2>/dev/null || (echo "$v $w FAILED"; tail -2 gpurun_out/$TAG/${v}_$w.err)
  done
done
