set -u
for c in "C2" "C3" "C3 --compact" "C4"; do
  n=$(echo $c | tr -d ' -'); timeout 900 python bench.py --config $c --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_$n.json 2> gpurun_out/bench_$n.err; echo "$c exit=$?"
  python -c "
import json;d=json.load(open('gpurun_out/bench_$n.json'));c=d['config'];print('$c tok/s %.3e ms %.1f step TB/s %.2f (%.0f%% of 8) fwd %.0f bwd %.0f' % (d['value'],d['ms_per_step'],c['achieved_hbm_gbs_step']/1e3,100*c['frac_of_8TBs_step'],c['fwd_sweep_gbs'],d['roofline']['achieved']))" || tail -3 gpurun_out/bench_$n.err
done
