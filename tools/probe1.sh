set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/p1_tests.txt
AB_SHAPES=qkv,o,gate_up,down,sq8192 timeout 300 python tools/mbs_ab.py > gpurun_out/p1_ab_pair.txt 2>&1
MXQ_MBS_CL=192 timeout 300 python tools/mbs_ab.py mbs_s > gpurun_out/p1_ab_192.txt 2>&1
cat gpurun_out/p1_*.txt
