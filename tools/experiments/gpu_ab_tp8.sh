# A/B on one box: vocabulary-shard rows (TP8 emulation) with the old vs new library
set -u
for r in 1 2; do for v in old new; do
  if [ $v = old ]; then export ESPO_LIB=$PWD/abtmp/libespo_old.so; else unset ESPO_LIB; fi
  timeout 600 python bench.py --vocab-shards 8 --no-e2e --no-cpu-baseline --no-factored-leg --steps 3 > gpurun_out/tp8_$v.json 2>/dev/null
  python -c "
import json;d=json.loads(open('gpurun_out/tp8_$v.json').read().strip().splitlines()[-1]);c=d['config'];print('$v', round(d['value']/1e6,3), 'M tok/s', round(d['ms_per_step'],1), 'ms; fwd', round(c['fwd_sweep_ms_per_chunk'],3), 'bwd', round(c['bwd_sweep_ms_per_chunk'],3), round(d['roofline']['achieved']), d['clocks']['sm_mhz'])"
done; done
timeout 600 python -m pytest tests/test_gpu_vocab_parallel.py -x -q > gpurun_out/vp.log 2>&1; echo vp=$?; tail -n 1 gpurun_out/vp.log
