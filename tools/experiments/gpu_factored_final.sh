# factored mode: full GPU suite, bench lines (C1, C3), traffic, one full ncu capture
set -u
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "gpu tests exit=$?"; tail -n 2 gpurun_out/gpu_tests.log
timeout 900 python bench.py --factored > gpurun_out/bench_C1factored.json 2> gpurun_out/bench_C1factored.err; echo "bench C1 factored exit=$?"
timeout 900 python bench.py --factored --config C3 --no-e2e --no-cpu-baseline > gpurun_out/bench_C3factored.json 2> gpurun_out/bench_C3factored.err; echo "bench C3 factored exit=$?"
timeout 900 python bench.py --factored --config C3 --compact --no-e2e --no-cpu-baseline > gpurun_out/bench_C3compact_factored.json 2> gpurun_out/bench_C3cf.err; echo "bench C3 compact factored exit=$?"
P="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --factored"
$P > gpurun_out/plain_ftr.log 2>&1 && ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:"k_fwd_grad|k_fwd_rows|k_row_scale" --csv --log-file gpurun_out/fact_traffic.csv $P > gpurun_out/ncu_ftr.log 2>&1; echo "traffic exit=$?"
Q="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --buffer-rows 8192 --factored"
$Q > gpurun_out/plain_fq.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"k_fwd_grad" -s 10 -c 1 -o gpurun_out/prof_factored $Q > gpurun_out/ncu_fact.log 2>&1; echo "ncu exit=$?"
