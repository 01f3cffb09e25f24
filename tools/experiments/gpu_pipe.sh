set -u
python -m pytest tests/test_gpu_parity.py -q -x -k "tiled_list" 2>&1 | tail -1
run() { n=$1; shift; timeout 600 python bench.py "$@" --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/pp_$n.json 2> gpurun_out/pp_$n.err;
python -c "
import json;d=json.load(open('gpurun_out/pp_$n.json'));c=d['config'];print('$n ms %.2f bwd %.0f' % (d['ms_per_step'],d['roofline']['achieved']))" || tail -3 gpurun_out/pp_$n.err; }
for r in 1 2; do for b in 10 12; do run C3c_b$b --config C3 --compact --bwd-impl $b; done; done
