#!/bin/bash
# ncu --set full of the row-prefetching instantiation (SCONV_WS_RP_FORCE=1: the one the density
# gate picks at s = 0.7) on conv1_2 (WsW PECR, the dominant launch) and conv4_2 (WsA), s = 0.7
mkdir -p gpurun_out
for L in conv1_2 conv4_2; do
SCONV_WS_RP_FORCE=1 S=0.7 LAYERS=$L LAYER_AB_CHILD=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:ecr_ws_kernel -c 1 -o gpurun_out/n_$L -f python tools/layer_ab.py > gpurun_out/n_${L}.log 2>&1; tail -1 gpurun_out/n_${L}.log
done
