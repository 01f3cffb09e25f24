# K2 ring geometries: deeper rings on 1/8- and 1/4-vocabulary shard rows and at full width
mkdir -p gpurun_out/r2am
for impl in 0 16 17 18 19 20 21 22 0 16; do timeout 300 python tools/tp_layout_probe.py 8 32768 7 $impl >> gpurun_out/r2am/layout.jsonl 2>> gpurun_out/r2am/err.log; done
for impl in 0 16 17 19 22; do timeout 300 python tools/tp_layout_probe.py 4 32768 5 $impl >> gpurun_out/r2am/layout.jsonl 2>> gpurun_out/r2am/err.log; done
for impl in 0 16 17 19 22 0; do timeout 300 python tools/tp_layout_probe.py 1 16384 5 $impl >> gpurun_out/r2am/layout.jsonl 2>> gpurun_out/r2am/err.log; done
