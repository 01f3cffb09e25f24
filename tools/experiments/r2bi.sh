# dW GEMM DRAM bytes / clock per variant (ncu, one launch each): default (N-groups of 8,
# A ef / B el / C ef), N-groups of 16, all-normal L2 policies, dW lockstep 8/2
mkdir -p gpurun_out/r2bi
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed
run() { timeout 300 ncu --metrics $M --clock-control none --csv -k regex:"k_umma_gemm2" -s 4 -c 1 python tools/lmhead_bwd_once.py 4096 8192 0 $2 $3 $4 > gpurun_out/r2bi/$1.csv 2>&1; }
run default -1 -1 -1
run n16 -1 1048576 -1
run allnormal -1 -1 0
run dwsync8 $((( (8 | (2<<16)) << 32 ))) -1 -1
timeout 300 ncu --metrics $M --clock-control none --csv -k regex:"nvjet" -s 2 -c 2 python tools/lmhead_bwd_once.py 4096 8192 1 > gpurun_out/r2bi/cublas.csv 2>&1
