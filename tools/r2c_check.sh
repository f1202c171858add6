#!/bin/bash
# round-2 session-3 check: GPU parity of the late bulk + SoA MDP sweep, A/B timings
T=${1:-r2c}; mkdir -p gpurun_out/$T
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/$T/tests.log 2>&1; echo "tests rc=$?"; grep -E "FAILED|Error|assert" gpurun_out/$T/tests.log | head -40; tail -3 gpurun_out/$T/tests.log
timeout 300 python tools/mdp_variants.py variants/m_pairs.so variants/m_soa.so variants/m_soa_u1.so variants/m_soa_i2f.so variants/m_soa512.so variants/m_soa512u1.so 2>&1 | tee gpurun_out/$T/mdp10k.txt
MDP_N=100000 timeout 300 python tools/mdp_variants.py variants/m_pairs.so variants/m_soa.so variants/m_soa512.so 2>&1 | tee gpurun_out/$T/mdp100k.txt
bash tools/odsvar.sh $T o_nobulk o_bulk 2>&1 | tee gpurun_out/$T/ods.txt
