#!/bin/bash
mkdir -p gpurun_out
A1=$PWD/paper_1909_09927_b200/lib_alt/libsconv_cuda.so
for S in 0.7 0.9; do
S=$S LAYERS=conv1_2,conv2_1,conv2_2,conv3_2,conv4_2,conv5_1 timeout 900 python tools/layer_ab.py "" "SCONV_LIB=$A1" > gpurun_out/pct2_$S.jsonl 2>&1
echo "s=$S"; python -c "
import json
for l in open('gpurun_out/pct2_$S.jsonl'):
    d=json.loads(l); print((d.get('variant') or 'default')[-24:], d.get('layer'), round(d.get('us',0)))
"
done
