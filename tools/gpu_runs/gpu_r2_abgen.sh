#!/bin/bash
# Generic layer A/B: variant 0 = $BASE_ENV (default: lib_alt = the previous build),
# then "" (this build) and each of $@.  SPARS / LAYERS select the sweep.
mkdir -p gpurun_out
A=$PWD/paper_1909_09927_b200/lib_alt/libsconv_cuda.so; A2=$PWD/paper_1909_09927_b200/lib_alt2/libsconv_cuda.so
BASE=${BASE_ENV:-SCONV_LIB=$A}
for S in ${SPARS:-0.7 0.9 0.95}; do
vars=("$BASE" "")
for v in "$@"; do vars+=("${v//@A2@/$A2}"); done
S=$S LAYERS=${LAYERS:-conv1_2,conv2_2,conv3_2,conv4_2,conv5_1} timeout 900 python tools/layer_ab.py "${vars[@]}" > gpurun_out/abgen_$S.jsonl 2>&1
echo "s=$S"; python - "$BASE" <<PY
import json, sys
base_v = sys.argv[1]
rows=[json.loads(l) for l in open('gpurun_out/abgen_$S.jsonl') if l.startswith('{')]
base={r['layer']:r['us'] for r in rows if r.get('variant')==base_v}
for r in rows:
    if r.get('variant') != base_v: print((r['variant'] or 'THIS')[-30:], r['layer'], 'base', round(base[r['layer']]), 'alt', round(r['us']), f"{(r['us']/base[r['layer']]-1)*100:+.1f}%", r.get("same_as_first"))
PY
done
