#!/bin/bash
# tools/build_mdp_variant.sh OUT.so -DSENECA_MDP_CHUNK=128 ...   (links against the in-tree capi/ods objects)
set -e
OUT=$1; shift
D=paper_2511_13724_b200
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr \
  -fmad=false -Iinclude "$@" -Xptxas -v -c $D/csrc/mdp.cu -o /tmp/mdp_variant_$$.o 2>&1 | grep -A2 "mdp_sweep_soa" | grep -E "Used|spill" | tr '\n' ' '; echo
nvcc -gencode arch=compute_100a,code=sm_100a -shared -Xcompiler -fPIC /tmp/mdp_variant_$$.o $D/_build/capi.o $D/_build/ods.o -o $OUT
rm -f /tmp/mdp_variant_$$.o
