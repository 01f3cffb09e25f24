set -u
python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -3
for r in 1 2; do for b in 0 8; do n=b${b}_$r; timeout 900 python bench.py --bwd-impl $b --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/x_$n.json 2> gpurun_out/x_$n.err;
python -c "
import json;d=json.load(open('gpurun_out/x_$n.json'));c=d['config'];print('$n ms %.2f step TB/s %.3f fwd %.0f (%.4f ms) bwd %.0f clk %s' % (d['ms_per_step'],c['achieved_hbm_gbs_step']/1e3,c['fwd_sweep_gbs'],c['fwd_sweep_ms_per_chunk'],d['roofline']['achieved'],d['clocks']['sm_mhz']))" || tail -5 gpurun_out/x_$n.err; done; done
