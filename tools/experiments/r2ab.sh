mkdir -p gpurun_out/r2ab
timeout 900 python -m pytest tests/test_gpu_lmhead.py tests/test_gpu_lmhead_fullsize.py tests/test_gpu_guard.py -q > gpurun_out/r2ab/test.log 2>&1; echo "rc=$?" >> gpurun_out/r2ab/test.log
M=gpu__time_duration.sum,dram__bytes_read.sum
timeout 600 ncu --metrics $M --clock-control none --cache-control none -k regex:"combine" --csv --log-file gpurun_out/r2ab/comb.csv python tools/lmhead_bwd_once.py 4096 8192 0 > /dev/null 2>&1
python tools/launch_table.py gpurun_out/r2ab/comb.csv 1 > gpurun_out/r2ab/comb.txt; rm gpurun_out/r2ab/comb.csv
timeout 900 python tools/bench_lmhead_fwd_ab.py 4096 3 4 > gpurun_out/r2ab/fwd_d4096.json 2> gpurun_out/r2ab/err.log
