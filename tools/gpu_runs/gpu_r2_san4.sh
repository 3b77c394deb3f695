#!/bin/bash
# round 2, pass 4: compute-sanitizer on the density-gated row-prefetch build (both
# ecr_ws_kernel instantiations, ws_density_gate_kernel); racecheck on the all-lanes
# build (lib_alt, -DSCONV_EMPTY_ALL_LANES=1, see profiles/r02/sanitizer.md)
mkdir -p gpurun_out
SEL="test_fixture_f5 or test_kats or test_ecr_fused or test_pecr_fused or test_smallc or test_ws_1x1_5x5 or test_ws_strided or test_pecr_other_pools or test_corrupted or test_all_zero or test_host_pointer_pipeline or (test_forced_kernels and (A or U or V or W or P))"
for tool in memcheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 --error-exitcode 9 \
     python -m pytest tests/test_gpu_parity.py -q -k "$SEL" -p no:cacheprovider > gpurun_out/san4_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/san4_$tool.log
  echo "$tool: $(grep -E 'ERROR SUMMARY|passed|failed|rc=' gpurun_out/san4_$tool.log | tr '\n' ' ')"
done
SCONV_LIB=$PWD/paper_1909_09927_b200/lib_alt/libsconv_cuda.so timeout 1500 compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 5 --error-exitcode 9 \
   python -m pytest tests/test_gpu_parity.py -q -k "test_ecr_fused or test_pecr_fused or test_ws_strided or (test_forced_kernels and (A or U or V or W))" -p no:cacheprovider > gpurun_out/san4_racecheck.log 2>&1
echo "rc=$?" >> gpurun_out/san4_racecheck.log
echo "racecheck (all-lanes build): $(grep -E 'RACECHECK SUMMARY|passed|failed|rc=' gpurun_out/san4_racecheck.log | tr '\n' ' ')"
