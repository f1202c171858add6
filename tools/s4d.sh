bash tools/odsab.sh s4d imagenet1k 3 base fast fast2
timeout 900 python -m pytest tests/test_gpu_ods.py -q -x > gpurun_out/s4d/ods_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/s4d/ods_tests.log
