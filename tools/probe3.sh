export AB_SHAPES=gate_up,sq8192
echo "== base"; timeout 300 python tools/mbs_ab.py mbs_s
for e in k1 k2 k3 k4 k7 k8 k16 k24; do echo "== $e"; MXQ_LIB_PATH=tools/_bin/libmxq200_$e.so timeout 300 python tools/mbs_ab.py mbs_s; done
