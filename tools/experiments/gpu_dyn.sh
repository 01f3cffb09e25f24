set -u
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_vocab_parallel.py -q -x 2>&1 | tail -2
for r in 1 2; do for v in old new; do
  if [ $v = old ]; then export ESPO_LIB=$PWD/abtmp/libespo_old.so; else unset ESPO_LIB; fi
  timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/dy.json 2>/dev/null
  python -c "
import json;d=json.load(open('gpurun_out/dy.json'));c=d['config'];print('$v C1 ms %.2f fwd %.0f bwd %.0f' % (d['ms_per_step'],c['fwd_sweep_gbs'],d['roofline']['achieved']))"
  timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --vocab-shards 8 > gpurun_out/dy8.json 2>/dev/null
  python -c "
import json;d=json.load(open('gpurun_out/dy8.json'));c=d['config'];print('$v TP8 ms %.2f fwd %.0f' % (d['ms_per_step'],c['fwd_sweep_gbs']))"
done; done
unset ESPO_LIB; timeout 300 python tools/experiments/tail_probe.py
