#!/bin/bash
# With the row prefetch in place: 2-tap cells (4 FFMA2 at R = 4) kept behind their branch
# (lib_g2: guard above 2 FFMA2 instead of 4) and no guard at all (lib_g0), vs this build
L=$PWD/paper_1909_09927_b200
BASE_ENV="SCONV_AB_BASE=1" SPARS="0.7 0.9" bash tools/gpu_runs/gpu_r2_abgen.sh "SCONV_LIB=$L/lib_g2/libsconv_cuda.so" "SCONV_LIB=$L/lib_g0/libsconv_cuda.so"
