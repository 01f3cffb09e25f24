# cuBLAS logits GEMM under the same ncu metrics as r2ao (d = 8192, 4096), and ours at g32
# with the soft lockstep on
mkdir -p gpurun_out/r2ap
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__throughput.avg.pct_of_peak_sustained_elapsed,lts__t_bytes.sum,launch__grid_size,launch__block_size,launch__cluster_dim_x
for d in 8192 4096; do
  timeout 300 ncu --metrics $M --clock-control none --csv -k regex:"nvjet|gemm|xmma|cutlass|sm100" -s 1 -c 1 python tools/lmhead_fwd_once.py $d 32768 -1 0 2 > gpurun_out/r2ap/d${d}_cublas.csv 2>&1
done
