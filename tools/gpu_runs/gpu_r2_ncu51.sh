#!/bin/bash
# ncu --set full of conv5_1 (14x14 maps, WsA) and conv2_1 (C = 64, persistent WsA) at s = 0.7
mkdir -p gpurun_out
for L in conv5_1 conv2_1; do
S=0.7 LAYERS=$L LAYER_AB_CHILD=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:ecr_ws -c 1 -o gpurun_out/n_$L -f python tools/layer_ab.py > gpurun_out/n_${L}.log 2>&1; tail -1 gpurun_out/n_${L}.log
done
