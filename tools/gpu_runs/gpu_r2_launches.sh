#!/bin/bash
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k 'regex:ecr_|pecr_|smallc|transpose|expand|pixel_nnz|ops_kernel|ws_density' -c 400 --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 1 --warmup 3 --no-cudnn --no-e2e --no-cpu --no-sweep --no-forward --no-check > gpurun_out/b_ncu.log 2>&1
tail -c 300 gpurun_out/b_ncu.log; wc -l gpurun_out/launches.csv
