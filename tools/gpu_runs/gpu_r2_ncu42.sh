#!/bin/bash
mkdir -p gpurun_out
S=0.7 LAYERS=conv4_2 LAYER_AB_CHILD=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:ecr_ws -c 1 -o gpurun_out/c42 -f python tools/layer_ab.py > gpurun_out/c42_ncu.log 2>&1; tail -1 gpurun_out/c42_ncu.log
S=0.7 LAYERS=conv1_2 LAYER_AB_CHILD=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:ecr_ws -c 1 -o gpurun_out/c12 -f python tools/layer_ab.py > gpurun_out/c12_ncu.log 2>&1; tail -1 gpurun_out/c12_ncu.log
