#!/bin/bash
# initcheck of pass 3 with the small-C kernel's STG epilogue (initcheck does not
# count TMA bulk-tensor stores as initialising writes)
mkdir -p gpurun_out
SEL="test_fixture_f5 or test_kats or test_ecr_fused or test_pecr_fused or test_smallc or test_ws_1x1_5x5 or test_ws_strided or test_pecr_other_pools or test_corrupted or test_all_zero or test_host_pointer_pipeline or (test_forced_kernels and (A or U or V or W or P))"
SCONV_SC2_STG=1 timeout 1500 compute-sanitizer --tool initcheck --print-limit 20 --error-exitcode 9 \
   python -m pytest tests/test_gpu_parity.py -q -k "$SEL" -p no:cacheprovider > gpurun_out/san3_initcheck_stg.log 2>&1
echo "rc=$?" >> gpurun_out/san3_initcheck_stg.log
echo "initcheck (STG epilogue): $(grep -E 'ERROR SUMMARY|passed|failed|rc=' gpurun_out/san3_initcheck_stg.log | tr '\n' ' ')"
