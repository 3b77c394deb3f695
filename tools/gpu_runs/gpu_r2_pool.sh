#!/bin/bash
# round 2: general-pool epilogue tests, the gpu suite, compute-sanitizer on small shapes
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -k "pecr_other_pools" -q > gpurun_out/pytest_pool.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_pool.log
tail -3 gpurun_out/pytest_pool.log
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
SEL="test_fixture_f5 or test_kats or test_ecr_fused or test_pecr_fused or test_smallc or test_ws_1x1_5x5 or test_ws_strided or test_pecr_other_pools or test_corrupted or test_all_zero or test_host_pointer_pipeline"
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 20 --error-exitcode 9 \
     python -m pytest tests/test_gpu_parity.py -q -k "$SEL" -p no:cacheprovider > gpurun_out/sanitizer_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/sanitizer_$tool.log
  tail -4 gpurun_out/sanitizer_$tool.log
done
