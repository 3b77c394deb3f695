#!/bin/bash
mkdir -p gpurun_out
S=0.7 LAYERS=conv1_2,conv2_1 timeout 900 python tools/layer_ab.py "" "SCONV_KERNEL=wC" "SCONV_KERNEL=wD" "SCONV_KERNEL=wE" "SCONV_KERNEL=wA" > gpurun_out/c12_ab.jsonl 2>&1
python -c "
import json
for l in open('gpurun_out/c12_ab.jsonl'):
    d=json.loads(l); print((d.get('variant') or 'default'), d.get('layer'), round(d.get('us',0)), d.get('error','')[:100])
"
