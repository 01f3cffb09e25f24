mkdir -p gpurun_out/r2i
timeout 900 python -m pytest tests/test_gpu_lmhead.py tests/test_gpu_lmhead_fullsize.py tests/test_gpu_guard.py -x -q > gpurun_out/r2i/test.log 2>&1; echo "rc=$?" >> gpurun_out/r2i/test.log
timeout 900 ncu --set full --clock-control none -k regex:"nvjet|umma_gemm2" -s 0 -c 4 -o gpurun_out/r2i/cmp_full python tools/gemm_sweep_pair.py > gpurun_out/r2i/ncu.log 2>&1
