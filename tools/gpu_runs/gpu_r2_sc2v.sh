#!/bin/bash
# conv1_1: small-C kernel variants (KG = 16; 8 rows per lane)
mkdir -p gpurun_out
A1=$PWD/paper_1909_09927_b200/lib_alt/libsconv_cuda.so; A2=$PWD/paper_1909_09927_b200/lib_alt2/libsconv_cuda.so
for lib in "" "$A1" "$A2"; do SCONV_LIB=$lib timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "smallc" 2>&1 | tail -1; done
LAYERS=conv1_1 timeout 600 python tools/layer_ab.py "" "SCONV_LIB=$A1" "SCONV_LIB=$A2" > gpurun_out/sc2v_ab.jsonl 2>&1; cat gpurun_out/sc2v_ab.jsonl
