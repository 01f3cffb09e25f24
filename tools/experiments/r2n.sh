mkdir -p gpurun_out/r2n
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__cycles_elapsed.avg.per_second,l1tex__m_xbar2l1tex_read_bytes_mem_global_op_tma_ld.sum
timeout 600 ncu --metrics $M --clock-control none --cache-control none --csv --log-file gpurun_out/r2n/launches_sync16.csv python tools/lmhead_bwd_once.py 4096 8192 0 16 > /dev/null 2>&1
timeout 600 ncu --metrics $M --clock-control none --cache-control none --csv --log-file gpurun_out/r2n/launches_sync4.csv python tools/lmhead_bwd_once.py 4096 8192 0 4 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --cache-control none -k regex:nvjet -s 0 -c 2 -o gpurun_out/r2n/nvjet_full python tools/lmhead_bwd_once.py 4096 8192 1 > gpurun_out/r2n/ncu.log 2>&1
