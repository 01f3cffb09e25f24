set -u
for r in 1 2; do for v in old new s1000; do
  case $v in old) export ESPO_LIB=$PWD/abtmp/libespo_old.so;; s1000) export ESPO_LIB=$PWD/abtmp/libespo_s1000.so;; new) unset ESPO_LIB;; esac
  timeout 120 python tools/lm_clock_probe.py 4096 > gpurun_out/sl.json 2>/dev/null
  python -c "
import json;d=json.load(open('gpurun_out/sl.json'));f=d['fused'];f2=d['fused2'];print('$v', 'fused %.0f TF/s @%s MHz %.0f W | again %.0f @%s' % (f['TFLOPs'], f['sm_mhz_median'], f['power_w_median'], f2['TFLOPs'], f2['sm_mhz_median']))"
done; done
