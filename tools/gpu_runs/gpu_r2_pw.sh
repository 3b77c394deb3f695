#!/bin/bash
# the pointwise (1x1) dense ordered GEMM: parity tests, then config 2 with it
# (this build) and without it (SCONV_NO_PW=1: the v3 1x1 configs)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "pointwise or ws_1x1_5x5" 2>&1 | tail -3
timeout 600 python tools/config2.py > gpurun_out/c2pw_on.jsonl 2> gpurun_out/c2pw_on.err
SCONV_NO_PW=1 timeout 600 python tools/config2.py > gpurun_out/c2pw_off.jsonl 2> gpurun_out/c2pw_off.err
python - <<'PY'
import json
on = {r['layer']: r for r in map(json.loads, open('gpurun_out/c2pw_on.jsonl'))}
off = {r['layer']: r for r in map(json.loads, open('gpurun_out/c2pw_off.jsonl'))}
for n, r in on.items():
    print(f"{n:26s} k{r['k']} kernel {r['kernel']} cudnn {r['cudnn_us']:7.1f}  pw {r['ours_us']:7.1f}  v3 {off[n]['ours_us']:7.1f}  exact {r['exact_bitwise_vs_oracle']}")
PY
