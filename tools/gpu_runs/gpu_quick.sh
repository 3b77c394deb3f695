#!/bin/bash
# Quick GPU iteration: micro (optional), gpu parity tests, per-layer probe.
mkdir -p gpurun_out
[ -n "$NOMICRO" ] || [ -x tools/micro/ffma2_rate.bin ] && timeout 120 tools/micro/ffma2_rate.bin > gpurun_out/micro.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python tools/probe_perf.py > gpurun_out/probe.txt 2>&1
tail -3 gpurun_out/pytest_gpu.log
cat gpurun_out/micro.txt gpurun_out/probe.txt
