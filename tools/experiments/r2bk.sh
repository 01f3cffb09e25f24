# dW L2 policies: A (dz panels shared by a wave's N-tiles) evict_last / normal, B (h) evict_last,
# C (fp32 read-add-write stream) evict_first; N-groups 8 and 16 — ncu DRAM / clock per launch
mkdir -p gpurun_out/r2bk
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed
# hints option: dW byte (bits 8-15) = A | B << 2 | C << 4 ; 1 ef, 2 el
H() { echo $(( ( $1 | ($2 << 2) | ($3 << 4) ) << 8 )); }
run() { timeout 300 ncu --metrics $M --clock-control none --csv -k regex:"k_umma_gemm2" -s 4 -c 1 python tools/lmhead_bwd_once.py 4096 8192 0 -1 $2 $3 > gpurun_out/r2bk/$1.csv 2>&1; }
run n8_ElElEf -1 $(H 2 2 1)
run n8_NoElEf -1 $(H 0 2 1)
run n16_ElElEf 1048576 $(H 2 2 1)
run n16_NoElEf 1048576 $(H 0 2 1)
run n4_ElElEf 262144 $(H 2 2 1)
