"""Dev: time forced kernel configs on VGG-shaped layers.
   KIDS=A,D LAYERS=conv3_2,conv4_2 python tools/ksweep.py"""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, paper_1909_09927_b200 as sc
ALL = {"conv1_2": (64, 64, 224), "conv2_1": (64, 128, 112), "conv2_2": (128, 128, 112),
       "conv3_1": (128, 256, 56), "conv3_2": (256, 256, 56), "conv4_1": (256, 512, 28),
       "conv4_2": (512, 512, 28), "conv5_1": (512, 512, 14)}
dev = torch.device("cuda:0")
S = float(os.environ.get("S", 0.7)); POOL = os.environ.get("POOL", "0") == "1"
def tm(fn, reps=5):
    for _ in range(2): fn()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    torch.cuda.synchronize(); e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3
kids = os.environ.get("KIDS", "0").split(",")
for name in os.environ.get("LAYERS", "conv3_2,conv4_2").split(","):
    C, K, H = ALL[name]
    g = torch.Generator(device=dev); g.manual_seed(1)
    x = torch.rand(64, C, H + 2, H + 2, device=dev, generator=g)
    x = x * (torch.rand(x.shape, device=dev, generator=g) >= S)
    w = torch.rand(K, C, 3, 3, device=dev, generator=g) - 0.5
    row = {"layer": name}
    for kid in kids:
        k = int(kid) if kid.isdigit() else kid
        try:
            if POOL:
                f = lambda: sc.pecr_conv_pool_batched(x, w, 1, sc.PoolConfig(2, 2, 2), fast=True, sync=False, kernel=k)
            else:
                f = lambda: sc.ecr_conv_batched(x, w, 1, fast=True, sync=False, kernel=k)
            row[kid] = round(tm(f), 1)
        except Exception as e:
            row[kid] = str(e)[:30]
    print(json.dumps(row), flush=True)
