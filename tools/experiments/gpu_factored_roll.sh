# rolling factored kernel (ESPO_OPT_FACTORED_IMPL 6-8) vs the default ring
set -u
timeout 900 python -m pytest tests/test_gpu_factored.py -x -q -k "impl or full_vocab" > gpurun_out/fact_tests.log 2>&1; echo "factored tests exit=$?"; tail -n 2 gpurun_out/fact_tests.log
B="python bench.py --no-e2e --no-cpu-baseline --no-factored-leg --steps 3"
for r in 1 2; do for v in 0 7 4 8; do
  timeout 600 $B --factored --factored-impl $v > gpurun_out/fv_$v.json 2> gpurun_out/fv_$v.err
  python - <<PY
import json
try:
    d = json.loads(open("gpurun_out/fv_$v.json").read().strip().splitlines()[-1])
    print("impl $v", "%.3f M tok/s" % (d["value"] / 1e6), "%.1f ms" % d["ms_per_step"], d["clocks"]["sm_mhz"])
except Exception as e:
    print("impl $v failed", e)
PY
done; done
P="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-factored-leg --factored --factored-impl 8"
$P > gpurun_out/plain_ftr.log 2>&1 && ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:"k_fwd_grad" -s 100 -c 4 --csv --log-file gpurun_out/fact_traffic8.csv $P > gpurun_out/ncu_ftr.log 2>&1; echo "traffic exit=$?"
