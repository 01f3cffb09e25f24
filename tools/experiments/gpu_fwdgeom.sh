set -u
run() { n=$1; shift; timeout 600 python bench.py "$@" --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/fg_$n.json 2> gpurun_out/fg_$n.err;
python -c "
import json;d=json.load(open('gpurun_out/fg_$n.json'));c=d['config'];print('$n ms %.2f fwd %.0f (%.4f ms) bwd %.0f clk %s' % (d['ms_per_step'],c['fwd_sweep_gbs'],c['fwd_sweep_ms_per_chunk'],d['roofline']['achieved'],d['clocks']['sm_mhz']))" || tail -3 gpurun_out/fg_$n.err; }
for f in 0 5 2 3 4 7 0 5 2 3 4 7; do run f$f --fwd-impl $f; done
