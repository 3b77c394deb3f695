"""Dev: conv1_1 (C=3, K=64, 224x224, N=64, s=0.7) under every forced config."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, paper_1909_09927_b200 as sc
dev = torch.device("cuda:0")
g = torch.Generator(device=dev); g.manual_seed(1)
C, K, H = int(os.environ.get("C", 3)), 64, 224
x = torch.rand(64, C, H + 2, H + 2, device=dev, generator=g)
x = x * (torch.rand(x.shape, device=dev, generator=g) >= 0.7)
w = torch.rand(K, C, 3, 3, device=dev, generator=g) - 0.5
def tm(fn, reps=10):
    for _ in range(3): fn()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    torch.cuda.synchronize(); e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3
out = {}
for kid in [0, 1, 2, 3, 4, 5, 6, 7, "A", "C", "D", "E", "F", "G"]:
    try:
        out[str(kid)] = round(tm(lambda: sc.ecr_conv_batched(x, w, 1, fast=True, sync=False, kernel=kid)), 1)
    except Exception as e:
        out[str(kid)] = str(e)[:40]
out["pool_default"] = round(tm(lambda: sc.pecr_conv_pool_batched(x, w, 1, sc.PoolConfig(2,2,2), fast=True, sync=False)), 1)
print(json.dumps(out))
