echo base; AB_SHAPES=qkv,o,gate_up,down,sq8192 timeout 200 python tools/mbs_ab.py mx16_oas,ocp32 2>&1 | sed 's/mbs_s.*TF\/s  mx16/mx16/'
echo bn192; MXQ_TC_BN=192 AB_SHAPES=qkv,o,gate_up,down,sq8192 timeout 200 python tools/mbs_ab.py mx16_oas,ocp32 2>&1
echo parity192; MXQ_TC_BN=192 timeout 600 python -m pytest tests/test_gpu_bench_parity.py -q -x -k "plain or bench_step" 2>&1 | tail -2
