"""Quick per-layer timing probe (dev tool; not the bench)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1909_09927_b200 as sc

VGG = [("conv1_1",3,64,224,0),("conv1_2",64,64,224,1),("conv2_1",64,128,112,0),("conv2_2",128,128,112,1),
       ("conv3_1",128,256,56,0),("conv3_2",256,256,56,0),("conv3_4",256,256,56,1),("conv4_1",256,512,28,0),
       ("conv4_2",512,512,28,0),("conv4_4",512,512,28,1),("conv5_1",512,512,14,0),("conv5_4",512,512,14,1)]
N = int(os.environ.get("N", 64)); S = float(os.environ.get("S", 0.7))
torch.backends.cudnn.allow_tf32 = False; torch.backends.cuda.matmul.allow_tf32 = False
torch.backends.cudnn.benchmark = True
dev = torch.device("cuda:0")
def tm(fn, reps=5):
    for _ in range(2): fn()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    torch.cuda.synchronize(); s.record()
    for _ in range(reps): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / reps * 1000
res = []
for name, C, K, Ho, pool in VGG:
    g = torch.Generator(device=dev); g.manual_seed(1)
    x = torch.rand(N, C, Ho + 2, Ho + 2, device=dev, generator=g)
    x = x * (torch.rand(x.shape, device=dev, generator=g) >= S)
    w = torch.rand(K, C, 3, 3, device=dev, generator=g) - 0.5
    nnz = (x != 0).float()
    # useful MACs = sum over windows nnz * K
    box = torch.nn.functional.conv2d(nnz.sum(1, keepdim=True), torch.ones(1,1,3,3,device=dev))
    macs = float(box.sum()) * K
    r = dict(layer=name)
    r["ecr_fast_us"] = tm(lambda: sc.ecr_conv_batched(x, w, 1, fast=True, sync=False))
    r["ecr_exact_us"] = tm(lambda: sc.ecr_conv_batched(x, w, 1, fast=False, sync=False))
    r["cudnn_us"] = tm(lambda: torch.nn.functional.conv2d(x, w))
    if pool:
        r["pecr_fast_us"] = tm(lambda: sc.pecr_conv_pool_batched(x, w, 1, sc.PoolConfig(2,2,2), fast=True, sync=False))
        r["cudnn_pool_us"] = tm(lambda: torch.nn.functional.max_pool2d(torch.relu(torch.nn.functional.conv2d(x, w)), 2))
    r["useful_tflops_fast"] = 2 * macs / r["ecr_fast_us"] / 1e6
    r["dense_tflops_cudnn"] = 2 * N * K * C * 9 * Ho * Ho / r["cudnn_us"] / 1e6
    # correctness spot-check vs cudnn
    y = sc.ecr_conv_batched(x, w, 1, fast=True)
    r["maxdiff_vs_cudnn"] = float((y - torch.nn.functional.conv2d(x, w)).abs().max())
    print(json.dumps(r), flush=True)
    res.append(r)
tot = {k: sum(r.get(k, 0) for r in res) for k in ("ecr_fast_us", "ecr_exact_us", "cudnn_us")}
print("TOTAL", json.dumps(tot))
