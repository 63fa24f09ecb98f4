timeout 300 ncu --set full --import-source on --clock-control none -k regex:k_nvfp4_runs -s 2 -c 1 -o gpurun_out/q3_nv python tools/profile_quant.py nvfp4 > gpurun_out/q_prof.log 2>&1
tail -2 gpurun_out/q_prof.log
