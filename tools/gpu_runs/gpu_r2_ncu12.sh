#!/bin/bash
# ncu --set full of conv1_2 (WsG PECR) and conv4_2 (WsA) at s = 0.7, current build
mkdir -p gpurun_out
for L in conv1_2 conv4_2; do
S=0.7 LAYERS=$L LAYER_AB_CHILD=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:ecr_ws -c 1 -o gpurun_out/n_$L -f python tools/layer_ab.py > gpurun_out/n_${L}.log 2>&1; tail -1 gpurun_out/n_${L}.log
done
