set -u
for d in 2048 4096 8192; do for cfg in "0 0" "0 1" "1 1" "2 1" "4 1" "8 1"; do set -- $cfg; timeout 300 python tools/bench_lmhead.py $d $1 $2 > gpurun_out/l2_${d}_${1}_${2}.json 2>&1; python -c "
import json;d=json.load(open('gpurun_out/l2_${d}_${1}_${2}.json'));print($d, 'parts', '$1', '2cta', $2, 'fused %.0f TF/s cublas %.0f' % (d['fused_lmhead_fwd']['TFLOPs'], d['cublas_matmul_bf16']['TFLOPs']))" || tail -2 gpurun_out/l2_${d}_${1}_${2}.json; done; done
