#!/bin/bash
T=${1:-r2o}; mkdir -p gpurun_out/$T
timeout 900 python -m pytest tests/test_gpu_ods.py -q -x > gpurun_out/$T/tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/$T/tests.log
bash tools/odsvar.sh $T o_nohoist o_hoist o_nohoist o_hoist 2>&1 | tee gpurun_out/$T/ods.txt
