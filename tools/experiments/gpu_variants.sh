# A/B of kernel variants on the legs where the default is weakest.
set -u
run() { n=$1; shift; timeout 900 python bench.py "$@" --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/var_$n.json 2> gpurun_out/var_$n.err; 
  python -c "
import json;d=json.load(open('gpurun_out/var_$n.json'));c=d['config'];print('$n ms %.1f step TB/s %.2f fwd %.0f bwd %.0f' % (d['ms_per_step'],c['achieved_hbm_gbs_step']/1e3,c['fwd_sweep_gbs'],d['roofline']['achieved']))" || tail -5 gpurun_out/var_$n.err; }
for b in 0 1 2 3 5; do run C3c_b$b --config C3 --compact --bwd-impl $b; done
for f in 0 1 2 5 7; do run tp8_f$f --vocab-shards 8 --fwd-impl $f; done
