set -u
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py -m gpu -q > gpurun_out/gpu_tests.log 2>&1; echo "gpu tests exit=$?"; tail -3 gpurun_out/gpu_tests.log
for a in "0 0" "2 0" "3 0" "5 0" "6 0" "0 5"; do set -- $a; timeout 400 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --fwd-impl $1 --bwd-impl $2 > gpurun_out/bench_$1$2.json 2> gpurun_out/bench_$1$2.err; python -c "
import json;d=json.load(open('gpurun_out/bench_$1$2.json'));c=d['config'];print('fwd $1 bwd $2: tok/s %.3e ms %.1f fwdGBs %.0f fwdms %.3f bwdms %.3f bwdGBs %.0f' % (d['value'],d['ms_per_step'],c['fwd_sweep_gbs'],c['fwd_sweep_ms_per_chunk'],c['bwd_sweep_ms_per_chunk'],d['roofline']['achieved']))" || tail -3 gpurun_out/bench_$1$2.err; done
