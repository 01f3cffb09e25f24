# factored-gradient geometry sweep (ESPO_OPT_FACTORED_IMPL) + DRAM traffic + one ncu capture
set -u
FI=${FI:-"0 2 3 4 5"}
NCU_IMPL=${NCU_IMPL:-0}
timeout 900 python -m pytest tests/test_gpu_factored.py -x -q > gpurun_out/fact_tests.log 2>&1; echo "factored tests exit=$?"; tail -n 3 gpurun_out/fact_tests.log
B="python bench.py --no-e2e --no-cpu-baseline --steps 3"
for r in 1 2; do
for v in $FI; do
  timeout 600 $B --factored --factored-impl $v > gpurun_out/fv_$v.json 2> gpurun_out/fv_$v.err
  python - <<PY
import json
try:
    d = json.loads(open("gpurun_out/fv_$v.json").read().strip().splitlines()[-1])
    print("impl $v", "%.3f M tok/s" % (d["value"] / 1e6), "%.1f ms" % d["ms_per_step"],
          "roof %.0f GB/s" % d["roofline"]["achieved"], d["clocks"]["sm_mhz"])
except Exception as e:
    print("impl $v failed", e)
PY
done; done
P="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --factored --factored-impl $NCU_IMPL"
$P > gpurun_out/plain_ftr.log 2>&1 && ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:"k_fwd_grad" -s 100 -c 6 --csv --log-file gpurun_out/fact_traffic.csv $P > gpurun_out/ncu_ftr.log 2>&1; echo "traffic exit=$?"
Q="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --buffer-rows 8192 --factored --factored-impl $NCU_IMPL"
$Q > gpurun_out/plain_fq.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"k_fwd_grad" -s 10 -c 1 -o gpurun_out/prof_fact_$NCU_IMPL $Q > gpurun_out/ncu_fact.log 2>&1; echo "ncu exit=$?"
