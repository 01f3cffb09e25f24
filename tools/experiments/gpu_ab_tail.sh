# A/B on one box: K2 skipping sub-batches past the row end (TP8 shard rows and C1)
set -u
for r in 1 2; do for v in old new; do
  if [ $v = old ]; then export ESPO_LIB=$PWD/abtmp/libespo_old.so; else unset ESPO_LIB; fi
  for leg in "--vocab-shards 8" ""; do
  timeout 600 python bench.py $leg --no-e2e --no-cpu-baseline --no-factored-leg --steps 3 > gpurun_out/ab_$v.json 2>/dev/null
  python -c "
import json;d=json.loads(open('gpurun_out/ab_$v.json').read().strip().splitlines()[-1]);c=d['config'];print('$v', '$leg', round(d['value']/1e6,3), 'M tok/s', round(d['ms_per_step'],1), 'ms; fwd', round(c['fwd_sweep_ms_per_chunk'],3), 'bwd', round(c['bwd_sweep_ms_per_chunk'],3), d['clocks']['sm_mhz'])"
  done
done; done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_vocab_parallel.py tests/test_gpu_single_pass.py tests/test_gpu_edges.py -x -q > gpurun_out/kt.log 2>&1; echo kt=$?; tail -n 1 gpurun_out/kt.log
