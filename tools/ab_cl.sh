#!/bin/bash
export PYTHONPATH=$PWD
for cl in 2 1; do echo "== CL=$cl"; MXQ_GEMM_CL=$cl timeout 100 python tools/gemm_timing.py; done
