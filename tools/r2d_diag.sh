#!/bin/bash
T=${1:-r2d}; mkdir -p gpurun_out/$T
python tools/wbw.py 2>&1 | tee gpurun_out/$T/wbw.txt
timeout 900 python bench.py > gpurun_out/$T/bench.json 2> gpurun_out/$T/bench.err; echo "bench rc=$?"; tail -3 gpurun_out/$T/bench.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ods_rounds -c 1 -o gpurun_out/$T/ods22k_early \
    python tools/profile_ods.py imagenet22k 8000 --plain > /dev/null 2>&1; echo "ncu rc=$?"
python tools/ncu_lines.py gpurun_out/$T/ods22k_early.ncu-rep 60 > gpurun_out/$T/lines_22k_early.txt 2>&1
python tools/ncu_lines.py gpurun_out/$T/ods22k_early.ncu-rep 60 --nobar > gpurun_out/$T/lines_22k_early_nobar.txt 2>&1
python tools/ncu_summary.py gpurun_out/$T/sum.md gpurun_out/$T/traffic.json ods22k_early=gpurun_out/$T/ods22k_early.ncu-rep > /dev/null 2>&1
ls -la gpurun_out/$T; rm -f gpurun_out/$T/*.ncu-rep
