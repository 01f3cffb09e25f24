set -u
run() { n=$1; shift; timeout 600 python bench.py "$@" --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/tg_$n.json 2> gpurun_out/tg_$n.err;
python -c "
import json;d=json.load(open('gpurun_out/tg_$n.json'));c=d['config'];print('$n ms %.2f fwd %.0f' % (d['ms_per_step'],c['fwd_sweep_gbs']))" || tail -3 gpurun_out/tg_$n.err; }
for r in 1 2; do for f in 0 2 3 4 7; do run tp8_f$f --vocab-shards 8 --fwd-impl $f; done; done
