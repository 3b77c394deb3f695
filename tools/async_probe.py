"""Dev: host-side timeline of asynchronous host-pointer calls over the VGG-19 layers."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, numpy as np
import paper_1909_09927_b200 as sc
from bench import VGG19, BATCH
xs, ws, ys = [], [], []
for l, (name, C, K, H, pooled) in enumerate(VGG19):
    x = torch.empty((BATCH, C, H + 2, H + 2), dtype=torch.float32, pin_memory=True)
    sc.generate_batch([l * 100 + n for n in range(BATCH)], H + 2, H + 2, C, 0.7, out=x.numpy())
    w = (torch.rand(K, C, 3, 3) - 0.5).pin_memory()
    oh = H // 2 if pooled else H
    xs.append(x.numpy()); ws.append(w.numpy())
    ys.append(torch.empty((BATCH, K, oh, oh), dtype=torch.float32, pin_memory=True).numpy())
pool = sc.PoolConfig(2, 2, 2)
def step(sync):
    marks = []
    t0 = time.perf_counter()
    for l, (name, C, K, H, pooled) in enumerate(VGG19):
        if pooled:
            sc.pecr_conv_pool_batched(xs[l], ws[l], 1, pool, fast=True, out=ys[l], sync=sync)
        else:
            sc.ecr_conv_batched(xs[l], ws[l], 1, fast=True, out=ys[l], sync=sync)
        marks.append(round((time.perf_counter() - t0) * 1e3, 1))
    sc.synchronize()
    return round((time.perf_counter() - t0) * 1e3, 1), marks
for mode in (True, False, False, False):
    tot, marks = step(mode)
    print("sync" if mode else "async", tot, "ms; host returns at", marks, flush=True)
