#!/bin/bash
# Window-row prefetch, chosen per launch by ws_density_gate_kernel (this build), forced off / on
# (SCONV_WS_RP_FORCE), vs the build before it (lib_alt); then the GPU test suite
L=$PWD/paper_1909_09927_b200
SPARS="${SPARS:-0.5 0.7 0.8 0.9 0.95}" bash tools/gpu_runs/gpu_r2_abgen.sh "SCONV_WS_RP_FORCE=0" "SCONV_WS_RP_FORCE=1"
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
