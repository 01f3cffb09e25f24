set -u
timeout 900 python bench.py > gpurun_out/sp_default.json 2> gpurun_out/sp_default.err; echo "default exit=$?"; cat gpurun_out/sp_default.json; tail -3 gpurun_out/sp_default.err
for c in "C1 --single-pass" "C3 --single-pass" "C1 --e2e-mode two-sweep"; do n=$(echo $c | tr -d ' -'); timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline $( [ "$c" = "C1 --e2e-mode two-sweep" ] || echo --no-e2e ) > gpurun_out/sp_$n.json 2> gpurun_out/sp_$n.err; echo "$c exit=$?"
python -c "
import json;d=json.load(open('gpurun_out/sp_$n.json'));c=d['config'];print('$n tok/s %.3e ms %.1f stepTB/s %.2f roof %.0f e2e %s' % (d['value'],d['ms_per_step'],c['achieved_hbm_gbs_step']/1e3,d['roofline']['achieved'], d['e2e'] and '%.3e' % d['e2e']['value']))" || tail -5 gpurun_out/sp_$n.err; done
