mkdir -p gpurun_out/r2ac
timeout 900 python -m pytest tests/test_gpu_lmhead.py -q -k "rlzvp" > gpurun_out/r2ac/test.log 2>&1; echo "rc=$?" >> gpurun_out/r2ac/test.log
