#!/bin/bash
T=${1:-r2q}; mkdir -p gpurun_out/$T
timeout 600 python -m pytest tests/test_gpu_mdp.py -q -x > gpurun_out/$T/tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/$T/tests.log
V="variants/m_pairs.so variants/m_ws.so variants/m_ws_u1.so"
timeout 300 python tools/mdp_variants.py $V 2>&1 | tee gpurun_out/$T/mdp10k.txt
MDP_N=100000 timeout 300 python tools/mdp_variants.py $V 2>&1 | tee gpurun_out/$T/mdp100k.txt
