# evictions pushed into the maintain CTA's shared memory (devq) vs dfill
mkdir -p gpurun_out/s4u
timeout 900 python -m pytest tests/test_gpu_ods.py -q -x > gpurun_out/s4u/t.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/s4u/t.log
bash tools/odsab.sh s4u imagenet1k 4 dfill devq
