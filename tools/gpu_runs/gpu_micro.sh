#!/bin/bash
mkdir -p gpurun_out
for b in tools/micro/*.bin; do echo "== $b"; timeout 120 $b; done > gpurun_out/micro.txt 2>&1
if [ -n "$NCU_LAYER" ]; then
LAYER=$NCU_LAYER POOL=${NCU_POOL:-0} timeout 600 ncu --set full --clock-control none --import-source on -k regex:ecr_ -s 2 -c 1 \
   -o gpurun_out/prof_q python tools/ncu_one.py > gpurun_out/ncu_q.log 2>&1
fi
cat gpurun_out/micro.txt
