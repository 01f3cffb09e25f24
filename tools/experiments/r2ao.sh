# LM-head forward on the GEMM core at d = 8192 / 4096: DRAM bytes, L2 hit rate, tensor-pipe
# activity and clock per raster group, next to cuBLAS (impl -1)
mkdir -p gpurun_out/r2ao
ncu --query-metrics 2>/dev/null | grep -i -E "tensor|pipe_tc|uma|utc" > gpurun_out/r2ao/metrics_avail.txt
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__throughput.avg.pct_of_peak_sustained_elapsed,lts__t_bytes.sum
for d in 8192 4096; do
  for g in 8 16 32 64 128; do
    timeout 300 ncu --metrics $M --clock-control none --csv -k regex:"k_umma_gemm|k_lmhead" -s 1 -c 1 python tools/lmhead_fwd_once.py $d 32768 0 $g 2 > gpurun_out/r2ao/d${d}_g$g.csv 2>&1
  done
  timeout 300 ncu --metrics $M --clock-control none --csv -k regex:"nvjet|gemm|sm100" -s 1 -c 1 python tools/lmhead_fwd_once.py $d 32768 -1 0 2 > gpurun_out/r2ao/d${d}_cublas.csv 2>&1
done
