set -u
true
for a in "0 7" "2 7" "4 7" "6 7" "1 7" "2 0"; do set -- $a; timeout 400 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --fwd-impl $1 --bwd-impl $2 > gpurun_out/bench_$1$2.json 2> gpurun_out/bench_$1$2.err; python -c "
import json;d=json.load(open('gpurun_out/bench_$1$2.json'));c=d['config'];print('fwd $1 bwd $2: tok/s %.3e ms %.1f fwdGBs %.0f fwdms %.3f bwdms %.3f bwdGBs %.0f' % (d['value'],d['ms_per_step'],c['fwd_sweep_gbs'],c['fwd_sweep_ms_per_chunk'],c['bwd_sweep_ms_per_chunk'],d['roofline']['achieved']))" || tail -3 gpurun_out/bench_$1$2.err; done
