mkdir -p gpurun_out/r2t
ESPO_DEBUG=1 timeout 600 python -m pytest "tests/test_gpu_lmhead.py::test_lmhead_bwd_matches_oracle" -x -q > gpurun_out/r2t/test.log 2>&1; echo "rc=$?" >> gpurun_out/r2t/test.log
