#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "ecr_fused or pecr_fused or forced or ws_ or vgg_full or pecr_other or host_pointer or determinism" > gpurun_out/bal_pytest.log 2>&1; tail -2 gpurun_out/bal_pytest.log
for S in 0.7 0.95; do
S=$S LAYERS=conv1_2,conv2_1,conv2_2,conv3_1,conv3_2,conv4_1,conv4_2,conv5_1,conv5_4 timeout 900 python tools/layer_ab.py "" "SCONV_WS_PACKED=1" > gpurun_out/bal_$S.jsonl 2>&1
echo "s=$S"; python -c "
import json
rows=[json.loads(l) for l in open('gpurun_out/bal_$S.jsonl')]
base={r['layer']:r['us'] for r in rows if r['variant']==''}
for r in rows:
    if r['variant']!='': print(r['layer'], 'balanced', round(base[r['layer']]), 'packed', round(r['us']), 'same', r['same_as_first'])
"
done
