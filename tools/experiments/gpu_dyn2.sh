set -u
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -1
for v in old new old new; do
  if [ $v = old ]; then export ESPO_LIB=$PWD/abtmp/libespo_old.so; else unset ESPO_LIB; fi
  timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --vocab-shards 8 > gpurun_out/dy8.json 2>/dev/null
  python -c "
import json;d=json.load(open('gpurun_out/dy8.json'));c=d['config'];print('$v TP8 ms %.2f fwd %.0f' % (d['ms_per_step'],c['fwd_sweep_gbs']))"
done
unset ESPO_LIB
timeout 600 python bench.py --config C3 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/dyc3.json 2>/dev/null; python -c "
import json;d=json.load(open('gpurun_out/dyc3.json'));c=d['config'];print('new C3 ms %.2f fwd %.0f' % (d['ms_per_step'],c['fwd_sweep_gbs']))"
