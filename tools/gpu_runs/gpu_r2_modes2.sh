#!/bin/bash
# EXACT-mode bench line and the config-5 (global batch 512 on one GPU) line
mkdir -p gpurun_out
timeout 900 python bench.py --exact --no-cpu --no-sweep --no-forward > gpurun_out/bench_exact.json 2> gpurun_out/bench_exact.err; tail -1 gpurun_out/bench_exact.err
timeout 1500 python bench.py --global-batch 512 --no-cpu --no-sweep --no-forward --no-cudnn > gpurun_out/bench_gb512.json 2> gpurun_out/bench_gb512.err; tail -1 gpurun_out/bench_gb512.err
python -c "
import json
for f in ('bench_exact', 'bench_gb512'):
    d = json.load(open(f'gpurun_out/{f}.json'))
    print(f, d['ms_per_step'], d['value'], d['config'].get('arith'), d['config'].get('global_batch'), d['e2e'] and d['e2e'].get('ms_per_step'))
"
