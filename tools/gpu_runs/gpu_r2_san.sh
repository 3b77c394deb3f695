#!/bin/bash
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python -m pytest tests/test_gpu_parity.py -q -x -k "smallc" > gpurun_out/san_$tool.log 2>&1
  echo "$tool: $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|passed|failed' gpurun_out/san_$tool.log | tr '\n' ' ')"
done
timeout 1500 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_export.py -q -x -k "pecr_export_device or scan" > gpurun_out/san_scan.log 2>&1
echo "scan memcheck: $(grep -E 'ERROR SUMMARY|passed|failed' gpurun_out/san_scan.log | tr '\n' ' ')"
