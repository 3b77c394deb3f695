#!/bin/bash
# A/B: default config vs the R = 8, 2x4-tile WsF on the C >= 128 VGG layers.
mkdir -p gpurun_out
for S in 0.7 0.95; do
S=$S LAYERS=conv2_2,conv3_1,conv3_2,conv4_2,conv5_1 timeout 900 python tools/layer_ab.py "" "SCONV_KERNEL=wF" > gpurun_out/wsf_$S.jsonl 2>&1
echo "s=$S"; python - <<PY
import json
rows=[json.loads(l) for l in open('gpurun_out/wsf_$S.jsonl') if l.startswith('{')]
base={r['layer']:r['us'] for r in rows if r.get('variant')==''}
for r in rows:
    if r.get('variant'): print(r['variant'], r['layer'], 'base', round(base[r['layer']]), 'alt', round(r['us']), f"{(r['us']/base[r['layer']]-1)*100:+.1f}%", r.get('same'))
PY
done
