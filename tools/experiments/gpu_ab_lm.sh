set -u
for r in 1 2; do for v in old new; do
  if [ $v = old ]; then export ESPO_LIB=$PWD/abtmp/libespo_old.so; else unset ESPO_LIB; fi
  for d in 4096 8192; do timeout 300 python tools/bench_lmhead.py $d > gpurun_out/ab_$d.json 2>&1; python -c "
import json;d=json.load(open('gpurun_out/ab_$d.json'));print('$v', $d, 'fused %.0f TF/s cublas %.0f' % (d['fused_lmhead_fwd']['TFLOPs'], d['cublas_matmul_bf16']['TFLOPs']))"; done
  timeout 300 python tools/bench_lmhead_bwd.py 4096 16384 > gpurun_out/abb.json 2>&1; python -c "
import json;d=json.load(open('gpurun_out/abb.json'));print('$v bwd', 'fused %.2f ms unfused %.2f ms bwd-only %.0f TF/s' % (d['fused']['ms'], d['unfused']['ms'], d['fused_bwd_only']['TFLOPs_3gemm']))"
done; done
