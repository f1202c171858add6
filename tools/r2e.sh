#!/bin/bash
T=${1:-r2e}; mkdir -p gpurun_out/$T
V="variants/m_pairs_base.so variants/m_pairs_old.so variants/m_pairs_plain.so variants/m_soa.so variants/m_soa_plain.so"
timeout 300 python tools/mdp_variants.py $V 2>&1 | tee gpurun_out/$T/mdp10k.txt
MDP_N=100000 timeout 300 python tools/mdp_variants.py $V 2>&1 | tee gpurun_out/$T/mdp100k.txt
