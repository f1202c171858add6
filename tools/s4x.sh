# speculated refill ids pushed into the job CTAs with their seen flags read during the wait (dspec) vs HEAD
mkdir -p gpurun_out/s4x
SENECA_LIB=$PWD/variants/dspec.so timeout 900 python -m pytest tests/test_gpu_ods.py -q -x > gpurun_out/s4x/t.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/s4x/t.log
bash tools/odsab.sh s4x imagenet1k 4 head dspec
