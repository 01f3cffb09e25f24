# TMA-reduce dW epilogue on by default: LM-head suites + sweeps + bench_lmhead_bwd
mkdir -p gpurun_out/r2bt
timeout 1500 python -m pytest tests/test_gpu_lmhead.py tests/test_gpu_lmhead_fullsize.py tests/test_gpu_guard.py tests/test_gpu_graph.py -q > gpurun_out/r2bt/test.log 2>&1; echo "rc=$?" >> gpurun_out/r2bt/test.log
timeout 1500 python tools/gemm_sweep.py 4096 8192 151936 3 6 red > gpurun_out/r2bt/red_d4096.json 2> gpurun_out/r2bt/err.log
timeout 1500 python tools/gemm_sweep.py 8192 8192 151936 2 4 red > gpurun_out/r2bt/red_d8192.json 2>> gpurun_out/r2bt/err.log
timeout 900 python tools/bench_lmhead_bwd.py 4096 16384 > gpurun_out/r2bt/lmbwd_dense.json 2>> gpurun_out/r2bt/err.log
timeout 900 python tools/bench_lmhead_bwd.py 4096 32768 realistic > gpurun_out/r2bt/lmbwd_real.json 2>> gpurun_out/r2bt/err.log
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__cycles_elapsed.avg.per_second
timeout 600 ncu --metrics $M --clock-control none --cache-control none --csv --log-file gpurun_out/r2bt/ll.csv python tools/lmhead_bwd_once.py 4096 8192 0 > /dev/null 2>&1
timeout 600 ncu --metrics $M --clock-control none --cache-control none --csv --log-file gpurun_out/r2bt/ll8.csv python tools/lmhead_bwd_once.py 8192 8192 0 > /dev/null 2>&1
python tools/launch_table.py gpurun_out/r2bt/ll.csv 20 > gpurun_out/r2bt/ll.txt 2>&1
python tools/launch_table.py gpurun_out/r2bt/ll8.csv 20 > gpurun_out/r2bt/ll8.txt 2>&1
rm -f gpurun_out/r2bt/*.csv
