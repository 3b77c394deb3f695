#!/bin/bash
mkdir -p gpurun_out
SCONV_SC2_STG=1 timeout 1500 compute-sanitizer --tool initcheck --print-limit 5 python -m pytest tests/test_gpu_parity.py -q -x -k "smallc" > gpurun_out/san_initcheck_stg.log 2>&1
echo "initcheck (STG epilogue): $(grep -E 'ERROR SUMMARY|passed|failed' gpurun_out/san_initcheck_stg.log | tr '\n' ' ')"
