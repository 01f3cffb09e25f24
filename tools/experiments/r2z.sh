mkdir -p gpurun_out/r2z
Q="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-factored-leg --vocab-shards 8"
timeout 900 ncu --section SourceCounters --section WarpStateStats --section SpeedOfLight --clock-control none --import-source on -k regex:"k_rowstats_tma" -s 40 -c 1 -o /tmp/tp8src $Q > gpurun_out/r2z/ncu.log 2>&1
python tools/ncu_source_top.py /tmp/tp8src.ncu-rep 45 > gpurun_out/r2z/tp8_source_top.txt 2>&1
Q2="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-factored-leg"
timeout 900 ncu --section SourceCounters --section WarpStateStats --section SpeedOfLight --clock-control none --import-source on -k regex:"k_rowstats_tma" -s 10 -c 1 -o /tmp/fullsrc $Q2 > gpurun_out/r2z/ncu2.log 2>&1
python tools/ncu_source_top.py /tmp/fullsrc.ncu-rep 45 > gpurun_out/r2z/full_source_top.txt 2>&1
ncu -i /tmp/tp8src.ncu-rep --page details --csv > gpurun_out/r2z/tp8_details.csv 2>&1
ncu -i /tmp/fullsrc.ncu-rep --page details --csv > gpurun_out/r2z/full_details.csv 2>&1
