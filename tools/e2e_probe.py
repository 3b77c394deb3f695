"""Dev: host-pointer (e2e) call time per layer vs its PCIe bytes."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1909_09927_b200 as sc
res = {"chunks": os.environ.get("SCONV_CHUNKS", "default")}
for name, C, K, H, pooled in [("conv1_2", 64, 64, 224, True), ("conv3_2", 256, 256, 56, False),
                              ("conv4_2", 512, 512, 28, False)]:
    x = torch.empty((64, C, H + 2, H + 2), dtype=torch.float32, pin_memory=True)
    sc.generate_batch([n for n in range(64)], H + 2, H + 2, C, 0.7, out=x.numpy())
    w = (torch.rand(K, C, 3, 3) - 0.5).pin_memory()
    oh = H // 2 if pooled else H
    y = torch.empty((64, K, oh, oh), dtype=torch.float32, pin_memory=True)
    f = (lambda: sc.pecr_conv_pool_batched(x.numpy(), w.numpy(), 1, sc.PoolConfig(2, 2, 2), fast=True, out=y.numpy())) if pooled else \
        (lambda: sc.ecr_conv_batched(x.numpy(), w.numpy(), 1, fast=True, out=y.numpy()))
    f()
    t = time.perf_counter()
    for _ in range(3):
        f()
    dt = (time.perf_counter() - t) / 3
    b_in, b_out = x.numel() * 4, y.numel() * 4
    res[name] = dict(ms=round(dt * 1e3, 2), in_mb=b_in >> 20, out_mb=b_out >> 20,
                     ideal_ms=round(max(b_in / 55.5e9, b_out / 57.2e9) * 1e3, 2))
print(json.dumps(res))
