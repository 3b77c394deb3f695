#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "ws_1x1 or forced" 2>&1 | tail -3
timeout 600 python tools/config2.py > gpurun_out/config2.jsonl 2>&1; cat gpurun_out/config2.jsonl
timeout 120 python tools/pcie_probe.py
