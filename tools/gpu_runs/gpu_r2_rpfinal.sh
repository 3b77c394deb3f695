#!/bin/bash
# Row prefetch gated at 15% density: GPU suite, the default bench line, the launch list,
# and the A/B at s = 0.8 / 0.85 / 0.9 (the threshold's neighbourhood) against the pre-change build
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -2 gpurun_out/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k 'regex:ecr_|pecr_|smallc|transpose|expand|pixel_nnz|ops_kernel|ws_density' -c 400 --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 1 --warmup 1 --no-cudnn --no-e2e --no-cpu --no-sweep --no-forward --no-check > gpurun_out/b_ncu.log 2>&1
SPARS="0.8 0.85 0.9" bash tools/gpu_runs/gpu_r2_abgen.sh "SCONV_WS_RP_FORCE=0" "SCONV_WS_RP_FORCE=1" > gpurun_out/rp6.txt 2>&1
echo done
