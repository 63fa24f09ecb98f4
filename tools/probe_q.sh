echo base; timeout 120 python tools/quant_timing.py 4096 2>/dev/null
for v in p1c4 p2c2 p2c8 p4c2 p1c8; do echo $v; MXQ_LIB_PATH=tools/_bin/libmxq200_$v.so timeout 120 python tools/quant_timing.py 4096 2>/dev/null | head -4; done
echo big; timeout 120 python tools/quant_timing.py 4096 14336 2>/dev/null
