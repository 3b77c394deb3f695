#!/bin/bash
mkdir -p gpurun_out
A1=$PWD/paper_1909_09927_b200/lib_alt/libsconv_cuda.so; A2=$PWD/paper_1909_09927_b200/lib_alt2/libsconv_cuda.so
for S in 0.7 0.9; do
S=$S LAYERS=conv2_1,conv2_2,conv3_1,conv3_2,conv4_2,conv5_1 timeout 900 python tools/layer_ab.py "" "SCONV_LIB=$A1" "SCONV_LIB=$A2" > gpurun_out/ring_$S.jsonl 2>&1
echo "s=$S"; python -c "
import json
rows=[json.loads(l) for l in open('gpurun_out/ring_$S.jsonl')]
base={r['layer']:r['us'] for r in rows if r.get('variant')==''}
for r in rows:
    if r.get('variant'): print(r['variant'][-22:], r['layer'], 'base', round(base[r['layer']]), 'alt', round(r['us']), f\"{(r['us']/base[r['layer']]-1)*100:+.1f}%\")
"
done
