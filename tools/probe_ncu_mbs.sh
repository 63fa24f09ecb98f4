# ncu --set full of the product MBS GEMM at 8192^3 (one launch), source counters
timeout 300 ncu --set full --import-source on --clock-control none -k regex:k_gemm_mbs -s 1 -c 1 -o gpurun_out/$1 python tools/profile_one.py 8192 mbs_h > gpurun_out/$1.log 2>&1
tail -3 gpurun_out/$1.log
