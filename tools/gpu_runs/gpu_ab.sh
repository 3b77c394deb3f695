#!/bin/bash
# Dev A/B: kcheck timings with the in-tree lib and with lib_alt (another build variant).
mkdir -p gpurun_out
LAYERS=${LAYERS:-conv1_2,conv3_2,conv4_2,conv5_1} timeout 300 python tools/kcheck.py
SCONV_LIB=$PWD/paper_1909_09927_b200/lib_alt/libsconv_cuda.so LAYERS=${LAYERS:-conv1_2,conv3_2,conv4_2,conv5_1} timeout 300 python tools/kcheck.py
LAYERS=${LAYERS:-conv1_2,conv3_2,conv4_2,conv5_1} timeout 300 python tools/kcheck.py
