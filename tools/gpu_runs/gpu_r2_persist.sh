#!/bin/bash
mkdir -p gpurun_out
SCONV_WS_PERSIST=1 timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_full.py -q -x -k "ecr_fused or pecr_fused or forced or ws_ or vgg_layer_full or pecr_other or host_pointer or determinism or multi_context" > gpurun_out/persist_pytest.log 2>&1; tail -2 gpurun_out/persist_pytest.log
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_full.py -q -x -k "ecr_fused or pecr_fused or forced or ws_ or vgg_layer_full or pecr_other" > gpurun_out/persist_pytest0.log 2>&1; tail -2 gpurun_out/persist_pytest0.log
for S in 0.7 0.95; do
S=$S LAYERS=conv1_2,conv2_1,conv2_2,conv3_1,conv3_2,conv4_1,conv4_2,conv5_1,conv5_4 timeout 900 python tools/layer_ab.py "" "SCONV_WS_PERSIST=1" > gpurun_out/persist_$S.jsonl 2>&1
echo "s=$S"; python -c "
import json
rows=[json.loads(l) for l in open('gpurun_out/persist_$S.jsonl')]
base={r['layer']:r['us'] for r in rows if r.get('variant')==''}
for r in rows:
    if r.get('variant'): print(r['layer'], 'base', round(base[r['layer']]), 'persist', round(r['us']), f\"{(r['us']/base[r['layer']]-1)*100:+.1f}%\", r['same_as_first'])
"
done
