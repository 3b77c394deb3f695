#!/bin/bash
# round 2: forced-config sweep across sparsities + the gpu suite
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
for S in 0.7 0.9 0.95; do
  S=$S KIDS=A,E,B,C,D,F,G,P LAYERS=conv2_2,conv3_2,conv4_2,conv5_1 timeout 600 python tools/ksweep.py >> gpurun_out/cfgsweep.jsonl 2>&1
  S=$S POOL=1 KIDS=C,D,G,E LAYERS=conv1_2,conv2_2 timeout 600 python tools/ksweep.py >> gpurun_out/cfgsweep_pool.jsonl 2>&1
done
