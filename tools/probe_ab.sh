#!/bin/bash
# A/B device timing of MBS GEMM variants (tools/build_variant.sh builds):
#   tools/probe_ab.sh tag1 tag2 ...   -> gpurun_out/ab.txt
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for r in 1 2; do
for v in "$@"; do
  echo "== $v (round $r)"
  MXQ_LIB_PATH=tools/_bin/libmxq200_$v.so timeout 300 python tools/mbs_ab.py mbs_s
done
done > gpurun_out/ab.txt 2>&1
cat gpurun_out/ab.txt
