"""Dev: small grids (batch-1 forward layers, small batches) under the 4x4 and
2x2-tile configs.  python tools/smallgrid.py"""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, paper_1909_09927_b200 as sc
dev = torch.device("cuda:0")
SHAPES = [(1, 64, 128, 112), (1, 128, 128, 112), (1, 128, 256, 56), (1, 256, 256, 56),
          (1, 256, 512, 28), (1, 512, 512, 28), (1, 512, 512, 14), (8, 512, 512, 14),
          (4, 256, 256, 56), (16, 512, 512, 14), (2, 512, 512, 28)]
def tm(fn, reps=20):
    for _ in range(3): fn()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    torch.cuda.synchronize(); e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3
if os.environ.get("SHAPES"):  # "n:C:K:H,..."
    SHAPES = [tuple(int(v) for v in t.split(":")) for t in os.environ["SHAPES"].split(",")]
KIDS = os.environ.get("KIDS", "A,B,E,P").split(",")
POOLS = (False, True) if os.environ.get("POOL", "1") == "1" else (False,)
for n, C, K, H in SHAPES:
    g = torch.Generator(device=dev); g.manual_seed(1)
    x = torch.rand(n, C, H + 2, H + 2, device=dev, generator=g)
    x = x * (torch.rand(x.shape, device=dev, generator=g) >= 0.7)
    w = torch.rand(K, C, 3, 3, device=dev, generator=g) - 0.5
    row = {"n": n, "C": C, "K": K, "H": H, "plan": sc.launch_plan(n, C, H + 2, H + 2, K, 3, 3, 1)["kernel"]}
    for pool in POOLS:
        for kid in KIDS:
            if pool and kid == "B":
                continue
            try:
                f = (lambda: sc.pecr_conv_pool_batched(x, w, 1, sc.PoolConfig(2, 2, 2), fast=True, sync=False, kernel=int(kid) if kid.isdigit() else kid)) if pool \
                    else (lambda: sc.ecr_conv_batched(x, w, 1, fast=True, sync=False, kernel=int(kid) if kid.isdigit() else kid))
                row[("p" if pool else "") + kid] = round(tm(f), 1)
            except Exception as e:
                row[("p" if pool else "") + kid] = str(e)[:20]
    print(json.dumps(row), flush=True)
