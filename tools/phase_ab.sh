# bash tools/phase_ab.sh TAG WORKLOAD ROUNDS REPEATS lib...: job 0's in-kernel phase cycles per variant
TAG=$1; W=$2; R=$3; N=$4; shift 4
mkdir -p gpurun_out/$TAG
for i in $(seq 1 $N); do
  for v in "$@"; do
    SENECA_LIB=$PWD/variants/$v.so timeout 300 python tools/profile_ods.py $W $R 2>/dev/null | head -1 | sed "s/^/$v $i /"
  done
done
