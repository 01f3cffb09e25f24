mkdir -p gpurun_out/r2d
timeout 900 python -m pytest tests/test_gpu_lmhead.py tests/test_gpu_lmhead_fullsize.py -x -q > gpurun_out/r2d/test.log 2>&1; echo "rc=$?" >> gpurun_out/r2d/test.log
timeout 600 python tools/bench_lmhead_bwd.py 4096 16384 > gpurun_out/r2d/bwd_d4096.json 2> gpurun_out/r2d/bwd_d4096.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__cycles_elapsed.avg.per_second --clock-control none --csv --log-file gpurun_out/r2d/launches_native.csv python tools/lmhead_bwd_once.py 4096 8192 0 > /dev/null 2>&1
