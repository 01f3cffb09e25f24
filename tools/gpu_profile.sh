# One profiling round on the GPU box: bench, launch list, traffic list, two full captures.
set -u
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke exit=$?"; tail -1 gpurun_out/smoke.log
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1; echo "gpu tests exit=$?"; tail -2 gpurun_out/gpu_tests.log
timeout 900 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo "bench exit=$?"
P="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-factored-leg"
$P > gpurun_out/plain_ll.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $P > gpurun_out/ncu_ll.log 2>&1; echo "launch list exit=$?"
$P > gpurun_out/plain_tr.log 2>&1 && ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:"k_rowstats|k_fwd_rows|k_dlogits|k_bwd_rows|k_bwd_recs" -s 768 --csv --log-file gpurun_out/traffic.csv $P > gpurun_out/ncu_tr.log 2>&1; echo "traffic exit=$?"
Q="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-factored-leg --buffer-rows 8192"
$Q > gpurun_out/plain_q.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"k_rowstats_tma" -s 60 -c 1 -o gpurun_out/prof_fwd $Q > gpurun_out/ncu_fwd.log 2>&1; echo "ncu fwd exit=$?"
$Q > gpurun_out/plain_q2.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"k_dlogits" -s 60 -c 2 -o gpurun_out/prof_bwd $Q > gpurun_out/ncu_bwd.log 2>&1; echo "ncu bwd exit=$?"
F="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --factored"
$F > gpurun_out/plain_fll.log 2>&1 && ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_factored.csv $F > gpurun_out/ncu_fll.log 2>&1; echo "factored launch list exit=$?"
$Q --factored > gpurun_out/plain_fq.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"k_fwd_grad" -s 10 -c 1 -o gpurun_out/prof_factored $Q --factored > gpurun_out/ncu_fact.log 2>&1; echo "ncu factored exit=$?"
# summarise on the box (ncu reports are large): the profiles/ tree comes back under gpurun_out/
python tools/make_profiles.py r1 > gpurun_out/make_profiles.log 2>&1; echo "make_profiles exit=$?"
rm -rf gpurun_out/profiles_new && cp -r profiles gpurun_out/profiles_new && rm -f gpurun_out/*.ncu-rep
