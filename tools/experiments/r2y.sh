mkdir -p gpurun_out/r2y
P="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-factored-leg --vocab-shards 8"
$P > gpurun_out/r2y/plain.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none --csv --log-file gpurun_out/r2y/launches_tp8.csv $P > gpurun_out/r2y/ncu.log 2>&1
python tools/launch_summary.py gpurun_out/r2y/launches_tp8.csv > gpurun_out/r2y/launches_tp8.md 2>&1
rm -f gpurun_out/r2y/launches_tp8.csv
