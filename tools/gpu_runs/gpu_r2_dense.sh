#!/bin/bash
mkdir -p gpurun_out
LAYERS=conv1_2,conv2_1,conv3_2,conv4_2,conv5_1 timeout 900 python tools/dense_gemm_probe.py > gpurun_out/dense_probe.jsonl 2>&1; cat gpurun_out/dense_probe.jsonl
