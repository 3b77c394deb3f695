#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_full.py -q -x -k "ecr_fused or pecr_fused or vgg_layer_full or host_pointer" 2>&1 | tail -1
for S in 0.7 0.9; do S=$S LAYERS=conv2_1 timeout 600 python tools/layer_ab.py "" "SCONV_KERNEL=wE" 2>&1 | cut -c1-120; done
