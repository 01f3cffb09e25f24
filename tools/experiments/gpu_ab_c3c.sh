# A/B on one box: C3 compact with the old vs new library (ESPO_LIB)
set -u
for r in 1 2 3; do for v in old new; do
  if [ $v = old ]; then export ESPO_LIB=$PWD/abtmp/libespo_old.so; else unset ESPO_LIB; fi
  timeout 600 python bench.py --config C3 --compact --no-e2e --no-cpu-baseline --no-factored-leg --steps 3 > gpurun_out/c3c_$v.json 2>/dev/null
  python -c "
import json;d=json.loads(open('gpurun_out/c3c_$v.json').read().strip().splitlines()[-1]);print('$v', round(d['value']/1e6,3), 'M tok/s', round(d['ms_per_step'],1), 'ms; bwd/chunk', round(d['config']['bwd_sweep_ms_per_chunk'],3), d['clocks']['sm_mhz'])"
done; done
