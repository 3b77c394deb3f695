#!/bin/bash
mkdir -p gpurun_out
S=0.7 LAYERS=conv3_2,conv4_2,conv5_1,conv5_4 timeout 1500 python tools/layer_ab.py "" "SCONV_KERNEL=wE" "SCONV_KERNEL=wD" "SCONV_KERNEL=wF" "SCONV_KERNEL=wB" "SCONV_KERNEL=wC" > gpurun_out/cfg_ab.jsonl 2>&1
python -c "
import json
for l in open('gpurun_out/cfg_ab.jsonl'):
    d=json.loads(l); print(d.get('variant') or 'default', d.get('layer'), round(d.get('us',0)), d.get('same_as_first'), d.get('error','')[:150])
"
