"""Launch one VGG-shaped ECR layer a few times (for ncu)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1909_09927_b200 as sc
C, K, Ho = [int(v) for v in os.environ.get("LAYER", "512,512,28").split(",")]
N = int(os.environ.get("N", 64)); S = float(os.environ.get("S", 0.7))
fast = os.environ.get("FAST", "1") == "1"
pool = os.environ.get("POOL", "0") == "1"
dev = torch.device("cuda:0")
x = torch.rand(N, C, Ho + 2, Ho + 2, device=dev)
x = x * (torch.rand(x.shape, device=dev) >= S)
w = torch.rand(K, C, 3, 3, device=dev) - 0.5
for _ in range(3):
    if pool:
        sc.pecr_conv_pool_batched(x, w, 1, sc.PoolConfig(2, 2, 2), fast=fast)
    else:
        sc.ecr_conv_batched(x, w, 1, fast=fast)
torch.cuda.synchronize()
