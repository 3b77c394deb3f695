#!/bin/bash
mkdir -p gpurun_out
for v in "" "SCONV_NO_SC2=1" "SCONV_SC2_STG=1"; do echo "variant: $v"; env $v timeout 300 python tools/pair_probe.py; done > gpurun_out/pair.log 2>&1
PAIR=conv5_4,conv1_2 timeout 300 python tools/pair_probe.py >> gpurun_out/pair.log 2>&1
cat gpurun_out/pair.log
