# LM-head backward: soft lockstep on the dW GEMM alone (dense sub-chunks, sustained sweep)
mkdir -p gpurun_out/r2ax
timeout 1500 python tools/gemm_sweep.py 4096 8192 151936 3 6 syncdw > gpurun_out/r2ax/sweep_d4096.json 2> gpurun_out/r2ax/err.log
timeout 1500 python tools/gemm_sweep.py 8192 8192 151936 2 4 syncdw > gpurun_out/r2ax/sweep_d8192.json 2>> gpurun_out/r2ax/err.log
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__cycles_elapsed.avg.per_second
timeout 600 ncu --metrics $M --clock-control none --csv -k regex:"k_umma_gemm2<1" --log-file gpurun_out/r2ax/dw_default.csv python tools/lmhead_bwd_once.py 4096 8192 0 > /dev/null 2>&1
