mkdir -p gpurun_out/r2l
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__cycles_elapsed.avg.per_second,l1tex__m_xbar2l1tex_read_bytes_mem_global_op_tma_ld.sum
timeout 600 ncu --metrics $M --clock-control none --cache-control none --csv --log-file gpurun_out/r2l/launches_cublas.csv python tools/lmhead_bwd_once.py 4096 8192 1 > /dev/null 2>&1
timeout 600 ncu --metrics $M --clock-control none --cache-control none --csv --log-file gpurun_out/r2l/launches_pair.csv python tools/lmhead_bwd_once.py 4096 8192 0 > /dev/null 2>&1
