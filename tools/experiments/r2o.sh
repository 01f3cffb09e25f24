mkdir -p gpurun_out/r2o
timeout 900 python -m pytest tests/test_gpu_lmhead.py tests/test_gpu_guard.py -x -q > gpurun_out/r2o/test.log 2>&1; echo "rc=$?" >> gpurun_out/r2o/test.log
timeout 900 python tools/gemm_sweep.py 4096 8192 151936 3 6 > gpurun_out/r2o/sweep_d4096_burst6.json 2> gpurun_out/r2o/err.log
timeout 900 python tools/gemm_sweep.py 8192 8192 151936 2 4 > gpurun_out/r2o/sweep_d8192_burst4.json 2>> gpurun_out/r2o/err.log
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__cycles_elapsed.avg.per_second,l1tex__m_xbar2l1tex_read_bytes_mem_global_op_tma_ld.sum
timeout 600 ncu --metrics $M --clock-control none --cache-control none --csv --log-file gpurun_out/r2o/launches_default.csv python tools/lmhead_bwd_once.py 4096 8192 0 > /dev/null 2>&1
timeout 600 ncu --metrics $M --clock-control none --cache-control none --csv --log-file gpurun_out/r2o/launches_pair512.csv python tools/lmhead_bwd_once.py 4096 8192 4 > /dev/null 2>&1
