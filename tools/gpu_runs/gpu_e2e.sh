#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "ws_1x1 or pipeline" 2>&1 | tail -1
timeout 300 python tools/e2e_probe.py
timeout 600 python bench.py --no-cudnn --no-cpu --no-forward > gpurun_out/bench_pipe.json 2> gpurun_out/bench_pipe.err
python -c "import json; d=json.load(open('gpurun_out/bench_pipe.json')); print('value', d['value'], 'ms', d['ms_per_step'], 'e2e', d['e2e']['ms_per_step'])"
