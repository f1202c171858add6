#!/bin/bash
# tools/build_ods_variant.sh OUT.so -DSENECA_ODS_THREADS=256 ...   (links against the in-tree capi/mdp objects)
set -e
OUT=$1; shift
D=paper_2511_13724_b200
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr \
  -Iinclude "$@" -Xptxas -v -c $D/csrc/ods.cu -o /tmp/ods_variant_$$.o 2>&1 | grep -A1 "ods_rounds" | grep -E "Used|spill" | tr '\n' ' '; echo
nvcc -gencode arch=compute_100a,code=sm_100a -shared -Xcompiler -fPIC /tmp/ods_variant_$$.o $D/_build/capi.o $D/_build/mdp.o -o $OUT
rm -f /tmp/ods_variant_$$.o
