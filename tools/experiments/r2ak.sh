# TP shard layout probe + the seeding test fix
mkdir -p gpurun_out/r2ak
timeout 600 python -m pytest tests/test_gpu_vocab_parallel.py -q > gpurun_out/r2ak/test.log 2>&1; echo "rc=$?" >> gpurun_out/r2ak/test.log
for impl in 0 2 4 5 7; do timeout 300 python tools/tp_layout_probe.py 8 32768 5 $impl >> gpurun_out/r2ak/layout.jsonl 2>> gpurun_out/r2ak/err.log; done
timeout 300 python tools/tp_layout_probe.py 2 32768 5 0 >> gpurun_out/r2ak/layout.jsonl 2>> gpurun_out/r2ak/err.log
