#!/bin/bash
# round 2: new tests first, full gpu suite, racecheck main vs all-lanes build, bench
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_full.py -k "pecr_other_pools or packed" -q > gpurun_out/pytest_new.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_new.log
tail -3 gpurun_out/pytest_new.log
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
SEL="test_ecr_fused or test_pecr_fused or test_ws_strided or test_pecr_other_pools"
for v in main alt; do
  if [ $v = alt ]; then export SCONV_LIB=$PWD/paper_1909_09927_b200/lib_alt/libsconv_cuda.so; fi
  timeout 1200 compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 5 \
     python -m pytest tests/test_gpu_parity.py -q -k "$SEL" -p no:cacheprovider > gpurun_out/racecheck_$v.log 2>&1
  echo "racecheck $v rc=$?" >> gpurun_out/racecheck_$v.log
  tail -3 gpurun_out/racecheck_$v.log
  unset SCONV_LIB
done
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -2 gpurun_out/bench.err
