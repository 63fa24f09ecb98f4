export AB_SHAPES=sq8192
timeout 300 python tools/mbs_ab.py mbs_s
for e in c1 k1 k1c1 k3 k3c1 k31 k31c1; do echo "== $e"; MXQ_LIB_PATH=tools/_bin/libmxq200_$e.so timeout 300 python tools/mbs_ab.py mbs_s; done
