mkdir -p gpurun_out/r2e
timeout 600 python -m pytest tests/test_gpu_lmhead.py -x -q > gpurun_out/r2e/test.log 2>&1; echo "rc=$?" >> gpurun_out/r2e/test.log
timeout 600 python tools/gemm_sweep.py 4096 8192 > gpurun_out/r2e/sweep_d4096.json 2> gpurun_out/r2e/sweep.err
timeout 600 python tools/gemm_sweep.py 8192 8192 > gpurun_out/r2e/sweep_d8192.json 2>> gpurun_out/r2e/sweep.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__cycles_elapsed.avg.per_second --clock-control none --csv --log-file gpurun_out/r2e/launches_cublas.csv python tools/lmhead_bwd_once.py 4096 8192 1 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__cycles_elapsed.avg.per_second --clock-control none --csv --log-file gpurun_out/r2e/launches_native.csv python tools/lmhead_bwd_once.py 4096 8192 0 > /dev/null 2>&1
