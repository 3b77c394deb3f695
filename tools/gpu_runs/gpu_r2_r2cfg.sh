#!/bin/bash
# A/B: WsA (4x4 tiles, R = 4) vs the R = 2 wide-tile configs on the C >= 128 layers
mkdir -p gpurun_out
for S in 0.95 0.9 0.7; do
S=$S LAYERS=conv3_2,conv4_2,conv5_1 timeout 900 python tools/layer_ab.py "" "SCONV_KERNEL=wC" "SCONV_KERNEL=wG" > gpurun_out/r2cfg_$S.jsonl 2>&1
echo "s=$S"; python - <<PY
import json
rows=[json.loads(l) for l in open('gpurun_out/r2cfg_$S.jsonl') if l.startswith('{')]
base={r['layer']:r['us'] for r in rows if r.get('variant')==''}
for r in rows:
    if r.get('variant'): print(r['variant'], r['layer'], 'base', round(base[r['layer']]), 'alt', round(r['us']), f"{(r['us']/base[r['layer']]-1)*100:+.1f}%")
PY
done
