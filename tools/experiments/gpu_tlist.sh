set -u
run() { n=$1; shift; timeout 600 python bench.py "$@" --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/tl_$n.json 2> gpurun_out/tl_$n.err;
python -c "
import json;d=json.load(open('gpurun_out/tl_$n.json'));c=d['config'];print('$n ms %.2f step %.3f fwd %.0f bwd %.0f clk %s' % (d['ms_per_step'],c['achieved_hbm_gbs_step']/1e3,c['fwd_sweep_gbs'],d['roofline']['achieved'],d['clocks']['sm_mhz']))" || tail -3 gpurun_out/tl_$n.err; }
for b in 9 10 11 0; do run C3c_b$b --config C3 --compact --bwd-impl $b; done
run C3_b10 --config C3 --bwd-impl 10
run C3_b0 --config C3
