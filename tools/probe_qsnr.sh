timeout 120 python tools/dq_qsnr_timing.py 2>&1 | tail -6
timeout 300 ncu --set full --import-source on --clock-control none -k regex:k_qsnr_nodes -s 2 -c 1 -o gpurun_out/qsnr_prof python tools/dq_qsnr_timing.py > /dev/null 2>&1
ls gpurun_out/qsnr_prof*
