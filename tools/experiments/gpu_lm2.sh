set -u
python -m pytest tests/test_gpu_lmhead.py -q -x 2>&1 | tail -3
for d in 2048 4096 8192; do timeout 300 python tools/bench_lmhead.py $d > gpurun_out/lm2_$d.json 2>&1; python -c "
import json;d=json.load(open('gpurun_out/lm2_$d.json'));print($d, 'fused %.0f TF/s cublas %.0f' % (d['fused_lmhead_fwd']['TFLOPs'], d['cublas_matmul_bf16']['TFLOPs']))"; done
for d in 2048 4096; do timeout 300 python tools/bench_lmhead_bwd.py $d 16384 > gpurun_out/lmb2_$d.json 2>&1; python -c "
import json;d=json.load(open('gpurun_out/lmb2_$d.json'));print($d, 'fused %.2f ms unfused %.2f ms bwd-only %.0f TF/s' % (d['fused']['ms'], d['unfused']['ms'], d['fused_bwd_only']['TFLOPs_3gemm']))"; done
