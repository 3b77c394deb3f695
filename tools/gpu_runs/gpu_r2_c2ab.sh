#!/bin/bash
# config-2 layers (tools/config2.py) with this build and the lib_alt / lib_alt2 builds
mkdir -p gpurun_out
for L in lib lib_alt lib_alt2; do
  SCONV_LIB=$PWD/paper_1909_09927_b200/$L/libsconv_cuda.so timeout 600 python tools/config2.py > gpurun_out/c2_$L.jsonl 2> gpurun_out/c2_$L.err
done
python - <<'PY'
import json
res = {L: {r['layer']: r for r in map(json.loads, open(f'gpurun_out/c2_{L}.jsonl'))} for L in ('lib', 'lib_alt', 'lib_alt2')}
for name, r in res['lib'].items():
    print(f"{name:26s} k{r['k']} cudnn {r['cudnn_us']:7.1f}  this {r['ours_us']:7.1f}  alt {res['lib_alt'][name]['ours_us']:7.1f}  alt2 {res['lib_alt2'][name]['ours_us']:7.1f}  exact {r['exact_bitwise_vs_oracle']} {res['lib_alt2'][name]['exact_bitwise_vs_oracle']}")
PY
