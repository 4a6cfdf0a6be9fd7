#!/bin/bash
# Tuning build: recompile fused_ws.cu with extra -D flags into build_alt/libwinofuse_alt_<tag>.so
# (the other objects come from build/).  usage: tools/build_alt.sh <tag> <flags...>
set -e
tag=$1; shift
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -Xptxas -v -diag-suppress 1886 "$@" \
  -c paper_1912_02165_b200/csrc/fused_ws.cu -o build_alt/fused_ws_$tag.o 2> build_alt/fused_ws_$tag.log
objs=$(ls build/*.o | grep -v fused_ws.o)
nvcc -gencode arch=compute_100a,code=sm_100a -shared $objs build_alt/fused_ws_$tag.o -o build_alt/libwinofuse_alt_$tag.so
grep -A2 "fused_ws_kernel" build_alt/fused_ws_$tag.log | grep -E "spill|registers" | sort | uniq -c
