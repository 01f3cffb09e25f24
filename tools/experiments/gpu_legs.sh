# Extra bench legs (one JSON line each): RL-ZVP mode on C3, vocabulary-parallel (8 shards) on C1.
set -u
run() { n=$1; shift; timeout 900 python bench.py "$@" --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_$n.json 2> gpurun_out/bench_$n.err; echo "$n exit=$?";
  python -c "
import json;d=json.load(open('gpurun_out/bench_$n.json'));c=d['config'];print('$n tok/s %.3e ms %.1f step TB/s %.2f fwd %.0f bwd %.0f launches %d' % (d['value'],d['ms_per_step'],c['achieved_hbm_gbs_step']/1e3,c['fwd_sweep_gbs'],d['roofline']['achieved'],d['gpu_launches']))" || tail -5 gpurun_out/bench_$n.err; }
run C3rlzvp --config C3 --zv-mode rlzvp
run C3mask --config C3
run C1tp8 --vocab-shards 8
run C1tp2 --vocab-shards 2
