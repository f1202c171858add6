#!/bin/bash
T=${1:-r2f}; mkdir -p gpurun_out/$T
./tools/micro/store_pattern 10000 | tee gpurun_out/$T/store10k.txt
./tools/micro/store_pattern 100000 | tee gpurun_out/$T/store100k.txt
timeout 900 python -m pytest tests/test_gpu_ods.py -q -x -k "storage_list or arrivals or launches or golden or toy or thirty" > gpurun_out/$T/tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/$T/tests.log
bash tools/odsvar.sh $T o_bulk o_bulk2 2>&1 | tee gpurun_out/$T/ods.txt
