#!/bin/bash
# GPU pass: parity tests then the default bench line.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
timeout 900 python bench.py "$@" > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -3 gpurun_out/bench.err
