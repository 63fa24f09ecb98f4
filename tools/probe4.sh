ncu --set full --clock-control none -k regex:k_gemm_mbs2 -s 1 -c 1 -o gpurun_out/p4_pair python tools/profile_one.py 8192 mbs_h > gpurun_out/p4_log1.txt 2>&1
MXQ_MBS_CL=192 ncu --set full --clock-control none -k regex:k_gemm_mbs -s 1 -c 1 -o gpurun_out/p4_192 python tools/profile_one.py 8192 mbs_h > gpurun_out/p4_log2.txt 2>&1
ncu --set full --clock-control none -k regex:k_gemm_tc -s 1 -c 1 -o gpurun_out/p4_ocp python tools/profile_one.py 8192 ocp32 > gpurun_out/p4_log3.txt 2>&1
ls -la gpurun_out
