# K2 reference seeding for rows without their target (vocabulary shards): tests, TP8 and C1
# bench lines, SASS blocks of the TP8 sweep
mkdir -p gpurun_out/r2aj
timeout 900 python -m pytest tests/test_gpu_vocab_parallel.py tests/test_gpu_parity.py tests/test_gpu_guard.py tests/test_gpu_edges.py tests/test_gpu_fullsize.py -q > gpurun_out/r2aj/test.log 2>&1; echo "rc=$?" >> gpurun_out/r2aj/test.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-factored-leg --vocab-shards 8 > gpurun_out/r2aj/tp8.json 2>/dev/null
timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-factored-leg --vocab-shards 2 > gpurun_out/r2aj/tp2.json 2>/dev/null
timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-factored-leg > gpurun_out/r2aj/c1.json 2>/dev/null
Q="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-factored-leg --buffer-rows 8192"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_rowstats_tma" -s 80 -c 1 -o gpurun_out/r2aj/tp8 $Q --vocab-shards 8 > gpurun_out/r2aj/ncu1.log 2>&1
python tools/ncu_summary.py gpurun_out/r2aj/tp8.ncu-rep > gpurun_out/r2aj/tp8_summary.txt 2>&1
ncu -i gpurun_out/r2aj/tp8.ncu-rep --page source --csv --print-source sass > gpurun_out/r2aj/tp8_sass.csv 2>&1
python tools/sass_blocks.py gpurun_out/r2aj/tp8_sass.csv 30 > gpurun_out/r2aj/tp8_blocks.txt 2>&1
rm -f gpurun_out/r2aj/*.ncu-rep gpurun_out/r2aj/*.csv
