#!/bin/bash
mkdir -p gpurun_out
ALT=$PWD/paper_1909_09927_b200/lib_alt/libsconv_cuda.so
for S in 0.95 0.9 0.7; do
  S=$S LAYERS=conv1_2,conv2_1,conv3_2,conv4_2,conv5_1 timeout 900 python tools/layer_ab.py "" "SCONV_LIB=$ALT" > gpurun_out/sparse_ab_$S.jsonl 2>&1
done
for S in 0.95 0.9 0.7; do echo "s=$S"; cat gpurun_out/sparse_ab_$S.jsonl | python -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l); print(d.get('variant','')[-20:], d.get('layer'), round(d.get('us',0)), d.get('same_as_first'), d.get('error','')[:200])
"; done
