#!/bin/bash
# Dev: ncu --set full of one forced-kernel launch per SCONV_KERNEL value (args).
mkdir -p gpurun_out
for k in "$@"; do
  SCONV_KERNEL=$k LAYER=${LAYER:-512,512,28} POOL=${POOL:-0} timeout 600 ncu --set full --clock-control none --import-source on \
    -k regex:${KREGEX:-ecr_} -s 2 -c 1 -o gpurun_out/prof_$k python tools/ncu_one.py > gpurun_out/ncu_$k.log 2>&1
  tail -2 gpurun_out/ncu_$k.log
done
