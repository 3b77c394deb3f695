#!/bin/bash
mkdir -p gpurun_out
for N in 48 56 57 60 64; do
  N=$N LAYERS=conv4_2,conv5_1,conv3_2 LAYER_AB_CHILD=1 timeout 600 python tools/layer_ab.py | sed "s/^/N=$N /"
done > gpurun_out/waves.log 2>&1
cat gpurun_out/waves.log
