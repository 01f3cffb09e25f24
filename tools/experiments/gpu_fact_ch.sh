# factored ring chunk size that divides a 152k-vocabulary row evenly (30 KB: 9.9 chunks)
set -u
B="python bench.py --no-e2e --no-cpu-baseline --no-factored-leg --steps 3"
for r in 1 2 3; do for v in 0 7 8; do
  timeout 600 $B --factored --factored-impl $v > gpurun_out/fv_$v.json 2> gpurun_out/fv_$v.err
  python -c "
import json;d=json.loads(open('gpurun_out/fv_$v.json').read().strip().splitlines()[-1]);print('impl $v', round(d['value']/1e6,3), 'M tok/s', round(d['ms_per_step'],1), d['clocks']['sm_mhz'])"
done; done
