#!/bin/bash
# Dev: host-pointer pipeline tests + e2e-only bench + config-2 layers.
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -k "pipeline or host or dropin or forward" 2>&1 | tail -2
timeout 600 python bench.py --no-cudnn --no-cpu --no-forward > gpurun_out/bench_pipe.json 2> gpurun_out/bench_pipe.err
python -c "import json; d=json.load(open('gpurun_out/bench_pipe.json')); print('value', d['value'], 'ms', d['ms_per_step'], 'e2e', d['e2e'])"
timeout 600 python tools/config2.py > gpurun_out/config2.jsonl 2>&1; cat gpurun_out/config2.jsonl
