set -u
timeout 900 python -m pytest tests/test_gpu_factored.py -x -q > gpurun_out/fact_tests.log 2>&1; echo "factored tests exit=$?"; tail -n 3 gpurun_out/fact_tests.log
B="python bench.py --no-e2e --no-cpu-baseline --steps 3"
for r in 1 2; do for v in 0 3 5 2; do
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
