#!/bin/bash
# EXACT-mode step and BASELINE config 5 (global batch 512) on one GPU
mkdir -p gpurun_out
timeout 900 python bench.py --exact --steps 5 --no-cudnn --no-e2e --no-cpu --no-sweep --no-forward > gpurun_out/bench_exact.json 2> gpurun_out/bench_exact.err; tail -c 400 gpurun_out/bench_exact.json; echo
timeout 1500 python bench.py --global-batch 512 --steps 3 --no-cudnn --no-cpu --no-sweep --no-forward > gpurun_out/bench_gb512.json 2> gpurun_out/bench_gb512.err; tail -c 400 gpurun_out/bench_gb512.json; echo
