#!/bin/bash
# Development variant of libmxq200.so with extra nvcc defines on the GEMM
# sources (the other objects are reused from the product build):
#   tools/build_variant.sh <tag> -DMXQ_MBS2_EXP=1 ...   -> tools/_bin/libmxq200_<tag>.so
set -e
tag=$1; shift
cd "$(dirname "$0")/.."
out=tools/_bin/var_$tag; mkdir -p $out
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -ftz=false -prec-div=true -prec-sqrt=true -fmad=true --expt-relaxed-constexpr $*"
L=paper_2603_08713_b200/_lib
objs="$L/capi.o $L/quantize.o $L/qsnr.o $L/layout.o $L/gemm_exact.o"
for s in gemm_tc gemm_mbs; do
  nvcc $F -c paper_2603_08713_b200/csrc/$s.cu -o $out/$s.o & objs="$objs $out/$s.o"
done
wait
nvcc -shared -gencode arch=compute_100a,code=sm_100a -o tools/_bin/libmxq200_$tag.so $objs -cudart static
echo tools/_bin/libmxq200_$tag.so
