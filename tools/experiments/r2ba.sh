# LM-head forward (d = 4096, default): full ncu capture with source — where do the MMA issuer
# and the producer wait (operand barriers vs accumulator-free barriers vs lockstep)?
mkdir -p gpurun_out/r2ba
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_umma_gemm" -s 1 -c 1 -o gpurun_out/r2ba/fwd python tools/lmhead_fwd_once.py 4096 32768 0 0 2 > gpurun_out/r2ba/ncu.log 2>&1
python tools/ncu_summary.py gpurun_out/r2ba/fwd.ncu-rep > gpurun_out/r2ba/summary.txt 2>&1
python tools/ncu_source_top.py gpurun_out/r2ba/fwd.ncu-rep 60 samples cuda > gpurun_out/r2ba/src_samp.txt 2>&1
ncu -i gpurun_out/r2ba/fwd.ncu-rep --page source --csv --print-source sass > gpurun_out/r2ba/sass.csv 2>&1
python tools/sass_blocks.py gpurun_out/r2ba/sass.csv 40 > gpurun_out/r2ba/blocks.txt 2>&1
rm -f gpurun_out/r2ba/*.ncu-rep
gzip -f gpurun_out/r2ba/sass.csv
