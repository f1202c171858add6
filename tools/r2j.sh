#!/bin/bash
T=${1:-r2j}; mkdir -p gpurun_out/$T
V="variants/m_base.so variants/m_g2.so variants/m_g1.so variants/m_w4.so variants/m_w4g2.so variants/m_w4g1.so"
timeout 300 python tools/mdp_variants.py $V 2>&1 | tee gpurun_out/$T/mdp10k.txt
MDP_N=100000 timeout 300 python tools/mdp_variants.py $V 2>&1 | tee gpurun_out/$T/mdp100k.txt
