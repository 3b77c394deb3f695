#!/bin/bash
# Dev: correctness + timing of several forced kernels (args = SCONV_KERNEL values).
mkdir -p gpurun_out
for k in "$@"; do SCONV_KERNEL=$k timeout 300 python tools/kcheck.py 2>&1 | tail -2; done | tee gpurun_out/kcheck.txt
