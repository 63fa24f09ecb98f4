MXQ_LIB_PATH=tools/_bin/libmxq200_tr1.so timeout 120 python tools/trace_skel.py > gpurun_out/p2_skel.txt 2>&1
MXQ_LIB_PATH=tools/_bin/libmxq200_tr2.so timeout 120 python tools/trace_mbs5.py > gpurun_out/p2_mbs5.txt 2>&1
cat gpurun_out/p2_*.txt
