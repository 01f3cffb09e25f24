# per-kernel times of the LM-head backward (native GEMMs vs cuBLAS), then full captures of
# the two native GEMM kernels
mkdir -p gpurun_out/r2c
timeout 300 python tools/lmhead_bwd_once.py 4096 8192 0 > gpurun_out/r2c/once.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file gpurun_out/r2c/launches_native.csv python tools/lmhead_bwd_once.py 4096 8192 0 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r2c/launches_cublas.csv python tools/lmhead_bwd_once.py 4096 8192 1 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_umma_gemm -s 0 -c 2 -o gpurun_out/r2c/gemm_full python tools/lmhead_bwd_once.py 4096 8192 0 > gpurun_out/r2c/ncu_full.log 2>&1
