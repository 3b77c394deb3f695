#!/bin/bash
mkdir -p gpurun_out
if [ -n "$TESTS" ]; then timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3; fi
timeout 900 python tools/tune.py "$@" > gpurun_out/tune.txt 2>&1
if [ -n "$S2" ]; then S=$S2 timeout 900 python tools/tune.py "$@" >> gpurun_out/tune.txt 2>&1; fi
cat gpurun_out/tune.txt
