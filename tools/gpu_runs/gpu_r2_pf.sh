#!/bin/bash
# A/B: next-channel mask prefetch (lib_pf), row prefetch (lib_rp), both (lib_both) vs the base build (lib_alt)
L=$PWD/paper_1909_09927_b200
SPARS="0.7 0.95" bash tools/gpu_runs/gpu_r2_abgen.sh "SCONV_LIB=$L/lib_pf/libsconv_cuda.so" "SCONV_LIB=$L/lib_rp/libsconv_cuda.so" "SCONV_LIB=$L/lib_both/libsconv_cuda.so"
