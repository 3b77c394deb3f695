import os, sys, numpy as np, torch
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import paper_1909_09927_b200 as sc
from oracle.oracle import c_oracle
orc = c_oracle()
N, C, K, size, s = 64, 480, 192, 14, 0.9
x = np.stack([orc.generate(size, size, C, s, 7_000_000 + n) for n in range(N)])
w = np.stack([orc.generate(1, 1, C, 0.0, 8_000_000 + j) for j in range(K)]) - np.float32(0.5)
xt, wt = torch.from_numpy(x).cuda(), torch.from_numpy(w).cuda()
for fast in (False, True):
    f = lambda: sc.ecr_conv_batched(xt, wt, 1, fast=fast, sync=False)
    for _ in range(3): f()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record()
    for _ in range(20): f()
    e1.record(); torch.cuda.synchronize()
    print("fast" if fast else "exact", round(e0.elapsed_time(e1) / 20 * 1e3, 1), "us")
