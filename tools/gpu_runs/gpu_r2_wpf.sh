#!/bin/bash
# With the row prefetch: the next channel's tap rows 0-1 read during the last two window rows (lib_wpf) vs this build
L=$PWD/paper_1909_09927_b200
BASE_ENV="SCONV_AB_BASE=1" SPARS="0.5 0.7 0.8" bash tools/gpu_runs/gpu_r2_abgen.sh "SCONV_LIB=$L/lib_wpf/libsconv_cuda.so"
