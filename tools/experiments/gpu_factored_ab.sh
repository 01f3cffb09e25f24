# A/B on one box: two-sweep default vs factored geometries
set -u
B="python bench.py --no-e2e --no-cpu-baseline --steps 3"
for r in 1 2 3; do
  for v in two 0 4 3; do
    if [ $v = two ]; then timeout 600 $B > gpurun_out/ab_$v.json 2> gpurun_out/ab_$v.err
    else timeout 600 $B --factored --factored-impl $v > gpurun_out/ab_$v.json 2> gpurun_out/ab_$v.err; fi
    python - <<PY
import json
d = json.loads(open("gpurun_out/ab_$v.json").read().strip().splitlines()[-1])
print("$v", "%.3f M tok/s" % (d["value"] / 1e6), "%.1f ms" % d["ms_per_step"], d["clocks"]["sm_mhz"], d["clocks"]["reasons"])
PY
  done
done
