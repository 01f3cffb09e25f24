mkdir -p gpurun_out/r2g
timeout 900 python -m pytest tests/test_gpu_guard.py -q > gpurun_out/r2g/test.log 2>&1; echo "rc=$?" >> gpurun_out/r2g/test.log
