# One profiling round on the GPU box: smoke, GPU tests, bench, launch list, traffic list, full
# captures (K2, K5, factored, K2 on TP8 shard rows, the LM-head backward's kernels), LM-head
# backward launch lists and A/B lines. usage: bash tools/gpu_profile.sh <tag>
set -u
TAG=${1:-r2}
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke exit=$?"; tail -1 gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1; echo "gpu tests exit=$?"; tail -2 gpurun_out/gpu_tests.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo "bench exit=$?"
timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-factored-leg --vocab-shards 8 > gpurun_out/bench_tp8.json 2>/dev/null; echo "tp8 exit=$?"
timeout 900 python bench.py --scaling strong --config C4 --steps 1 --warmup 3 --verify --no-e2e --no-cpu-baseline --no-factored-leg > gpurun_out/bench_C4_strong_verify.json 2>/dev/null; echo "c4 strong exit=$?"
for n in 2 4 8; do timeout 600 python bench.py --scaling strong --emulate-ranks $n --steps 5 --warmup 3 --verify > gpurun_out/bench_C1_emulate$n.json 2>/dev/null; echo "emulate $n exit=$?"; done
timeout 600 python bench.py --scaling strong --steps 5 --warmup 3 --verify --no-e2e --no-cpu-baseline --no-factored-leg > gpurun_out/bench_C1_strong_verify.json 2>/dev/null; echo "c1 strong exit=$?"
timeout 900 python bench.py --scaling strong --config C4 --emulate-ranks 8 --steps 1 --warmup 3 --verify > gpurun_out/bench_C4_emulate8.json 2>/dev/null; echo "c4 emulate8 exit=$?"
P="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-factored-leg"
$P > gpurun_out/plain_ll.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $P > gpurun_out/ncu_ll.log 2>&1; echo "launch list exit=$?"
# traffic: skip the 3 warm-up steps (C1 at 65,536-row chunks: 32 calls × 4 kernels per step)
$P > gpurun_out/plain_tr.log 2>&1 && ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:"k_rowstats|k_fwd_rows|k_dlogits|k_bwd_rows|k_bwd_recs" -s 384 --csv --log-file gpurun_out/traffic.csv $P > gpurun_out/ncu_tr.log 2>&1; echo "traffic exit=$?"
Q="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-factored-leg --buffer-rows 8192"
$Q > gpurun_out/plain_q.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"k_rowstats_tma" -s 60 -c 1 -o gpurun_out/prof_fwd $Q > gpurun_out/ncu_fwd.log 2>&1; echo "ncu fwd exit=$?"
$Q > gpurun_out/plain_q2.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"k_dlogits" -s 60 -c 2 -o gpurun_out/prof_bwd $Q > gpurun_out/ncu_bwd.log 2>&1; echo "ncu bwd exit=$?"
$Q --vocab-shards 8 > gpurun_out/plain_q3.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"k_rowstats_tma" -s 80 -c 1 -o gpurun_out/prof_tp8 $Q --vocab-shards 8 > gpurun_out/ncu_tp8.log 2>&1; echo "ncu tp8 exit=$?"
F="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --factored"
$F > gpurun_out/plain_fll.log 2>&1 && ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_factored.csv $F > gpurun_out/ncu_fll.log 2>&1; echo "factored launch list exit=$?"
$Q --factored > gpurun_out/plain_fq.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"k_fwd_grad" -s 10 -c 1 -o gpurun_out/prof_factored $Q --factored > gpurun_out/ncu_fact.log 2>&1; echo "ncu factored exit=$?"
# LM head backward: A/B lines, launch lists (native and cuBLAS), full captures of its kernels
timeout 900 python tools/bench_lmhead_bwd.py 4096 16384 > gpurun_out/bench_lmhead_bwd_dense.json 2>/dev/null; echo "lmhead bwd dense exit=$?"
timeout 900 python tools/bench_lmhead_bwd.py 4096 32768 realistic > gpurun_out/bench_lmhead_bwd_realistic.json 2>/dev/null; echo "lmhead bwd realistic exit=$?"
timeout 900 python tools/gemm_sweep.py 4096 8192 151936 3 6 > gpurun_out/gemm_sweep.json 2>/dev/null; echo "gemm sweep exit=$?"
timeout 900 python tools/bench_lmhead_fwd_ab.py 4096 3 4 default2 > gpurun_out/bench_lmhead_fwd_d4096.json 2>/dev/null; echo "lmhead fwd 4096 exit=$?"
timeout 900 python tools/bench_lmhead_fwd_ab.py 8192 2 3 default2 > gpurun_out/bench_lmhead_fwd_d8192.json 2>/dev/null; echo "lmhead fwd 8192 exit=$?"
MF=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,lts__t_bytes.sum
for d in 4096 8192; do timeout 300 ncu --metrics $MF --clock-control none --csv -k regex:"k_umma_gemm" -s 1 -c 1 python tools/lmhead_fwd_once.py $d 32768 0 0 2 > gpurun_out/ncu_lmhead_fwd_d$d.csv 2>&1; echo "ncu lmhead fwd $d exit=$?"; done
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__cycles_elapsed.avg.per_second
timeout 600 ncu --metrics $M --clock-control none --cache-control none --csv --log-file gpurun_out/launches_lmhead_bwd.csv python tools/lmhead_bwd_once.py 4096 8192 0 > /dev/null 2>&1; echo "lm ll exit=$?"
timeout 600 ncu --metrics $M --clock-control none --cache-control none --csv --log-file gpurun_out/launches_lmhead_bwd_cublas.csv python tools/lmhead_bwd_once.py 4096 8192 1 > /dev/null 2>&1; echo "lm ll cublas exit=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_umma_gemm" -s 0 -c 2 -o gpurun_out/prof_gemm python tools/lmhead_bwd_once.py 4096 8192 0 > gpurun_out/ncu_gemm.log 2>&1; echo "ncu gemm exit=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_lmhead_dz" -s 0 -c 1 -o gpurun_out/prof_lmdz python tools/lmhead_bwd_once.py 4096 8192 0 > gpurun_out/ncu_lmdz.log 2>&1; echo "ncu lmdz exit=$?"
# summarise on the box (ncu reports are large): the profiles/ tree comes back under gpurun_out/
python tools/make_profiles.py $TAG > gpurun_out/make_profiles.log 2>&1; echo "make_profiles exit=$?"
du -sh gpurun_out; ls -la gpurun_out/*.ncu-rep 2>/dev/null | head -20
rm -rf gpurun_out/profiles_new && cp -r profiles gpurun_out/profiles_new && rm -f gpurun_out/*.ncu-rep
find gpurun_out -type f -size +20M -print -delete
