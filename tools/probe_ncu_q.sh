timeout 300 ncu --set full --import-source on --clock-control none -k regex:k_quant_runs -s 3 -c 1 -o gpurun_out/q2_mx16 python tools/profile_quant.py mx16 > gpurun_out/q_prof.log 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:k_quant_runs -s 3 -c 1 -o gpurun_out/q2_mbss python tools/profile_quant.py mbs_s >> gpurun_out/q_prof.log 2>&1
tail -3 gpurun_out/q_prof.log
