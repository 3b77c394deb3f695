#!/bin/bash
# The bench's multi-rank path (torchrun, 2 ranks) exercised on a 1-GPU box:
# gloo for the barriers / max-over-ranks, both ranks on cuda:0 (timings share
# the device, so the numbers are not results -- the path is what is checked)
mkdir -p gpurun_out
export SCONV_BENCH_DIST=gloo
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 \
  bench.py --gpus 2 --steps 3 --warmup 3 --no-cudnn --no-cpu --no-sweep --no-forward > gpurun_out/mr_weak.json 2> gpurun_out/mr_weak.err
echo "weak rc=$? lines=$(wc -l < gpurun_out/mr_weak.json)"; tail -2 gpurun_out/mr_weak.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 \
  bench.py --gpus 2 --steps 3 --warmup 3 --global-batch 128 --no-cudnn --no-cpu --no-sweep --no-forward > gpurun_out/mr_strong.json 2> gpurun_out/mr_strong.err
echo "strong rc=$? lines=$(wc -l < gpurun_out/mr_strong.json)"; tail -2 gpurun_out/mr_strong.err
