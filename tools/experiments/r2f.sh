mkdir -p gpurun_out/r2f
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 300 python tools/sanitize_target.py > gpurun_out/r2f/plain.log 2>&1; echo "rc=$?" >> gpurun_out/r2f/plain.log
for tool in memcheck synccheck racecheck; do
  for part in c0 c1 lmhead tp; do
    ( time timeout 900 $CS --tool $tool --print-limit 10 --error-exitcode 9 python tools/sanitize_target.py $part ) > gpurun_out/r2f/${tool}_${part}.log 2>&1
    echo "rc=$?" >> gpurun_out/r2f/${tool}_${part}.log
  done
done
