# factored-gradient mode: tests, bench legs vs the default, DRAM traffic of k_fwd_grad
set -u
timeout 900 python -m pytest tests/test_gpu_factored.py -x -q > gpurun_out/fact_tests.log 2>&1; echo "factored tests exit=$?"; tail -3 gpurun_out/fact_tests.log
B="python bench.py --no-e2e --no-cpu-baseline"
for r in 1 2; do
  timeout 600 $B > gpurun_out/fact_def_$r.json 2> gpurun_out/fact_def_$r.err; echo "default exit=$?"
  timeout 600 $B --factored > gpurun_out/fact_$r.json 2> gpurun_out/fact_$r.err; echo "factored exit=$?"
  python - <<PY
import json
for n in ("fact_def_$r", "fact_$r"):
    try:
        d = json.loads(open(f"gpurun_out/{n}.json").read().strip().splitlines()[-1])
        print(n, "%.3f M tok/s" % (d["value"] / 1e6), "%.1f ms" % d["ms_per_step"],
              "roof %.0f GB/s" % d["roofline"]["achieved"], d["clocks"]["sm_mhz"])
    except Exception as e:
        print(n, "failed", e)
PY
done
P="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --factored"
$P > gpurun_out/plain_ftr.log 2>&1 && ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:"k_fwd_grad|k_fwd_rows" -s 200 -c 12 --csv --log-file gpurun_out/fact_traffic.csv $P > gpurun_out/ncu_ftr.log 2>&1; echo "traffic exit=$?"
