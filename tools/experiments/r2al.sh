# K2 ring geometries on 1/8-vocabulary shard rows (contiguous shard, 32768 rows)
mkdir -p gpurun_out/r2al
timeout 600 python -m pytest tests/test_gpu_vocab_parallel.py -q > gpurun_out/r2al/test.log 2>&1; echo "rc=$?" >> gpurun_out/r2al/test.log
for impl in 0 12 13 14 15 16 4 0; do timeout 300 python tools/tp_layout_probe.py 8 32768 7 $impl >> gpurun_out/r2al/layout.jsonl 2>> gpurun_out/r2al/err.log; done
for impl in 0 12 14; do timeout 300 python tools/tp_layout_probe.py 4 32768 5 $impl >> gpurun_out/r2al/layout.jsonl 2>> gpurun_out/r2al/err.log; done
