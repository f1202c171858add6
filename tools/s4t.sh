# DSMEM release carrying the refill split + ids pushed into job shared memory (dfill) vs DSMEM signals only (dsig)
mkdir -p gpurun_out/s4t
timeout 900 python -m pytest tests/test_gpu_ods.py -q -x > gpurun_out/s4t/t.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/s4t/t.log
bash tools/odsab.sh s4t imagenet1k 4 dsig dfill
