mkdir -p gpurun_out
for b in tools/micro/*.bin; do echo "== $b"; timeout 120 $b; done > gpurun_out/micro.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python tools/probe_perf.py > gpurun_out/probe.txt 2>&1
tail -3 gpurun_out/pytest_gpu.log
