set -u
for r in 1 2 3; do for v in old new; do
  if [ $v = old ]; then export ESPO_LIB=$PWD/abtmp/libespo_old.so; else unset ESPO_LIB; fi
  timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ab.json 2>/dev/null
  python -c "
import json;d=json.load(open('gpurun_out/ab.json'));c=d['config'];print('$v ms %.2f fwd %.0f bwd %.0f clk %s' % (d['ms_per_step'],c['fwd_sweep_gbs'],d['roofline']['achieved'],d['clocks']['sm_mhz']))"
done; done
