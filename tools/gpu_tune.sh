#!/bin/bash
mkdir -p gpurun_out
timeout 900 python tools/tune.py "$@" > gpurun_out/tune.txt 2>&1
cat gpurun_out/tune.txt
