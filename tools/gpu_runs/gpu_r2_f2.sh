#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_export.py tests/test_dropin.py tests/test_gpu_parity.py -q -m gpu > gpurun_out/f2_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/f2_pytest.log
tail -15 gpurun_out/f2_pytest.log
