#!/bin/bash
# GPU round-1 evidence pass: gpu tests, bench, launch list, one ncu --set full.
set -x
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvsmi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
   python bench.py --steps 1 --warmup 0 --no-cudnn --no-e2e --no-cpu > gpurun_out/bench_ncu.log 2>&1
LAYER=512,512,28 timeout 600 ncu --set full --clock-control none --import-source on -k regex:ecr_ -s 2 -c 1 \
   -o gpurun_out/prof_conv4 python tools/ncu_one.py > gpurun_out/ncu_full.log 2>&1
LAYER=64,64,224 POOL=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:ecr_ -s 2 -c 1 \
   -o gpurun_out/prof_conv1_2p python tools/ncu_one.py >> gpurun_out/ncu_full.log 2>&1
ls -la gpurun_out
