#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_full.py tests/test_forward.py tests/test_dropin.py -q -m gpu > gpurun_out/exact_pytest.log 2>&1; tail -2 gpurun_out/exact_pytest.log
timeout 900 python bench.py --exact --steps 5 --no-cudnn --no-e2e --no-cpu --no-sweep --no-forward > gpurun_out/bench_exact.json 2> gpurun_out/bench_exact.err; python -c "
import json; d=json.loads(open('gpurun_out/bench_exact.json').read().strip().splitlines()[-1]); print('exact ms/step', d['ms_per_step'])"
