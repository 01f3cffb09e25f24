mkdir -p gpurun_out/r2ad
ESPO_DEBUG=1 timeout 600 python -m pytest tests/test_gpu_lmhead.py -x -q -k "mcast or gemm_mc" > gpurun_out/r2ad/test.log 2>&1; echo "rc=$?" >> gpurun_out/r2ad/test.log
