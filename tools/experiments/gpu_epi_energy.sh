set -u
for r in 1 2; do for v in real noop; do
  if [ $v = noop ]; then export ESPO_LIB=$PWD/abtmp/libespo_noop.so; else unset ESPO_LIB; fi
  timeout 120 python tools/lm_clock_probe.py 4096 > gpurun_out/ee.json 2>/dev/null
  python -c "
import json;d=json.load(open('gpurun_out/ee.json'));f=d['fused'];c=d['cublas'];print('$v', 'fused %.0f TF/s @%s MHz %.0f W | cublas %.0f @%s MHz %.0f W' % (f['TFLOPs'], f['sm_mhz_median'], f['power_w_median'], c['TFLOPs'], c['sm_mhz_median'], c['power_w_median']))"
done; done
