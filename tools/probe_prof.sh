# (1) launch list of the bench command (kernel durations, cold-cache serialized under ncu)
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/r02_launches.csv python bench.py --steps 2 --warmup 3 --no-experts > gpurun_out/r02_bench_under_ncu.txt 2>&1
# (2) traffic + pipes of the four MBS-H layer GEMMs
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_write.sum,lts__t_sectors_srcunit_tex_op_read.sum,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed,smsp__issue_active.avg.pct_of_peak_sustained_active,l1tex__m_xbar2l1tex_read_bytes.sum --clock-control none -k regex:k_gemm -s 4 -c 4 --csv --log-file gpurun_out/r02_gemm_traffic_mbs.csv python tools/profile_layers.py mbs_h > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_write.sum,sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:k_gemm -s 4 -c 4 --csv --log-file gpurun_out/r02_gemm_traffic_ocp.csv python tools/profile_layers.py ocp32 > /dev/null 2>&1
# (3) full capture of the gate_up MBS GEMM with source counters
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_gemm_mbs -s 6 -c 1 -o gpurun_out/r02_mbs_gate_up python tools/profile_layers.py mbs_h > /dev/null 2>&1
ls -la gpurun_out | tail -8
