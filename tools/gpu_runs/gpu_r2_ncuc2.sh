#!/bin/bash
# ncu --set full of two config-2 layers (one launch each, FAST timing loop)
mkdir -p gpurun_out
for L in GoogLeNet.inception4a.1 GoogLeNet.inception5a.2; do
ONLY=$L N=64 timeout 600 ncu --set full --clock-control none --import-source on -k regex:ecr_ws --launch-skip 3 -c 1 -o gpurun_out/c2_$L -f python tools/config2.py > gpurun_out/c2n_$L.log 2>&1; tail -1 gpurun_out/c2n_$L.log
done
