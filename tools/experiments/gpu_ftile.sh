set -u
python -m pytest tests/test_gpu_parity.py -q -x -k "tiled_fwd" 2>&1 | tail -3
run() { n=$1; shift; timeout 600 python bench.py "$@" --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ft_$n.json 2> gpurun_out/ft_$n.err;
python -c "
import json;d=json.load(open('gpurun_out/ft_$n.json'));c=d['config'];print('$n ms %.2f step %.3f fwd %.0f (%.4f ms) bwd %.0f clk %s' % (d['ms_per_step'],c['achieved_hbm_gbs_step']/1e3,c['fwd_sweep_gbs'],c['fwd_sweep_ms_per_chunk'],d['roofline']['achieved'],d['clocks']['sm_mhz']))" || tail -3 gpurun_out/ft_$n.err; }
for f in 0 9 10 11 0; do run f$f --fwd-impl $f; done
