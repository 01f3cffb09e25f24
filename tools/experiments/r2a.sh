set -x
mkdir -p gpurun_out/r2a
python -m pytest tests -m gpu -x -q > gpurun_out/r2a/gputest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2a/gputest.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2a/bench_c1.json 2> gpurun_out/r2a/bench_c1.err
timeout 900 python bench.py --scaling strong --config C4 --steps 1 --warmup 3 --verify --no-e2e --no-cpu-baseline --no-factored-leg > gpurun_out/r2a/bench_c4_strong.json 2> gpurun_out/r2a/bench_c4_strong.err
timeout 600 python bench.py --scaling strong --config C1 --steps 5 --warmup 3 --verify --no-e2e --no-cpu-baseline --no-factored-leg > gpurun_out/r2a/bench_c1_strong.json 2> gpurun_out/r2a/bench_c1_strong.err
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-factored-leg --drift-seq 0.01 > gpurun_out/r2a/bench_c1_drift001.json 2> gpurun_out/r2a/bench_c1_drift001.err
