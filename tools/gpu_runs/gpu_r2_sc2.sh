#!/bin/bash
# smallc2 (lanes-over-pixels small-C ECR) A/B + parity + ncu
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "smallc" > gpurun_out/sc2_pytest.log 2>&1; tail -3 gpurun_out/sc2_pytest.log
ALT=$PWD/paper_1909_09927_b200/lib_alt/libsconv_cuda.so; LAYERS=conv1_1 timeout 600 python tools/layer_ab.py "" "SCONV_NO_SC2=1" "SCONV_LIB=$PWD/paper_1909_09927_b200/lib_alt/libsconv_cuda.so" > gpurun_out/sc2_ab.jsonl 2>&1; cat gpurun_out/sc2_ab.jsonl
LAYERS=conv1_1 LAYER_AB_CHILD=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:smallc2 -c 1 -o gpurun_out/sc2 -f python tools/layer_ab.py > gpurun_out/sc2_ncu.log 2>&1; tail -2 gpurun_out/sc2_ncu.log
