mkdir -p gpurun_out/r2x
ESPO_DEBUG=1 timeout 900 python -m pytest tests/test_gpu_lmhead.py -q -k "degenerate" > gpurun_out/r2x/test.log 2>&1; echo "rc=$?" >> gpurun_out/r2x/test.log
