set -u
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
run() { n=$1; shift; timeout 600 python bench.py "$@" --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/nd_$n.json 2> gpurun_out/nd_$n.err;
python -c "
import json;d=json.load(open('gpurun_out/nd_$n.json'));c=d['config'];print('$n ms %.2f step %.3f fwd %.0f bwd %.0f' % (d['ms_per_step'],c['achieved_hbm_gbs_step']/1e3,c['fwd_sweep_gbs'],d['roofline']['achieved']))" || tail -3 gpurun_out/nd_$n.err; }
run C1
run C1old --fwd-impl 5
run C1tp8 --vocab-shards 8
run C1tp8old --vocab-shards 8 --fwd-impl 5
run C3 --config C3
run C3old --config C3 --fwd-impl 5
