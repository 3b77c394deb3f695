#!/bin/bash
# ncu --set full of conv4_2 (WsA) at s = 0.7 and 0.95 with the current build
mkdir -p gpurun_out
for S in 0.7 0.95; do
S=$S LAYERS=conv4_2 LAYER_AB_CHILD=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:ecr_ws -c 1 -o gpurun_out/c42_$S -f python tools/layer_ab.py > gpurun_out/c42_${S}_ncu.log 2>&1; tail -1 gpurun_out/c42_${S}_ncu.log
done
