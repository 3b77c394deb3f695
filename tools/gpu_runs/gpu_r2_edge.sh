#!/bin/bash
# config U (half-tile edge bodies): parity + conv5 timing vs WsA
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_full.py -q -x -k "forced or edge_tiles or vgg_layer_full_size" > gpurun_out/edge_pytest.log 2>&1; tail -2 gpurun_out/edge_pytest.log
S=0.7 LAYERS=conv5_1,conv5_4,conv4_2 timeout 600 python tools/layer_ab.py "" "SCONV_NO_EDGE=1" > gpurun_out/edge_ab.jsonl 2>&1; cat gpurun_out/edge_ab.jsonl | cut -c1-160
