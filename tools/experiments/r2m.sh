mkdir -p gpurun_out/r2m
timeout 900 python tools/gemm_sweep.py 4096 8192 151936 3 6 > gpurun_out/r2m/sweep_d4096_burst6.json 2> gpurun_out/r2m/err.log
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__cycles_elapsed.avg.per_second
