# d = 8192 backward under the dynamic scheduler: tile / group variants + per-kernel launch lists
mkdir -p gpurun_out/r2bp
timeout 1500 python tools/gemm_sweep.py 8192 8192 151936 2 4 wide > gpurun_out/r2bp/wide_d8192.json 2> gpurun_out/r2bp/err.log
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__cycles_elapsed.avg.per_second
timeout 600 ncu --metrics $M --clock-control none --cache-control none --csv --log-file gpurun_out/r2bp/ll_native.csv python tools/lmhead_bwd_once.py 8192 8192 0 > /dev/null 2>&1
timeout 600 ncu --metrics $M --clock-control none --cache-control none --csv --log-file gpurun_out/r2bp/ll_cublas.csv python tools/lmhead_bwd_once.py 8192 8192 1 > /dev/null 2>&1
python tools/launch_table.py gpurun_out/r2bp/ll_native.csv 20 > gpurun_out/r2bp/ll_native.txt 2>&1
python tools/launch_table.py gpurun_out/r2bp/ll_cublas.csv 20 > gpurun_out/r2bp/ll_cublas.txt 2>&1
rm -f gpurun_out/r2bp/*.csv
