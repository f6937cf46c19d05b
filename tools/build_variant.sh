#!/bin/bash
# Build an experimental copy of libcorr2d.so with extra -D flags into _variants/
# (git-ignored, travels to the GPU box).  Usage: tools/build_variant.sh NAME -DFOO=1 ...
set -e
name=$1; shift
cd "$(dirname "$0")/.."
out=_variants/$name; mkdir -p $out
objs=()
for src in paper_1808_00685_b200/csrc/*.cu; do
  o=$out/$(basename ${src%.cu}).o
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xptxas -v "$@" \
    -I include -c $src -o $o 2> $out/$(basename ${src%.cu}).ptxas.txt &
  objs+=($o)
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o _variants/libcorr2d_$name.so "${objs[@]}" -cudart static
grep -A2 "2sm_kernelILi1" $out/contract_tc.ptxas.txt | grep -E "registers|spill" | head -2
echo _variants/libcorr2d_$name.so
