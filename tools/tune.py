"""Sweep the tiled-kernel configs (SCONV_TILED_CFG) over VGG-shaped layers."""
import json, os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import os, sys, json
sys.path.insert(0, %r)
import torch, paper_1909_09927_b200 as sc
N = int(os.environ.get("N", 64)); S = float(os.environ.get("S", 0.7))
dev = torch.device("cuda:0")
def tm(fn, reps=5):
    for _ in range(2): fn()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    torch.cuda.synchronize(); s.record()
    for _ in range(reps): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / reps * 1000
out = {}
for name, C, K, Ho in [("conv1_1",3,64,224),("conv1_2",64,64,224),("conv2_2",128,128,112),("conv3_2",256,256,56),("conv4_2",512,512,28),("conv5_1",512,512,14)]:
    g = torch.Generator(device=dev); g.manual_seed(1)
    x = torch.rand(N, C, Ho + 2, Ho + 2, device=dev, generator=g)
    x = x * (torch.rand(x.shape, device=dev, generator=g) >= S)
    w = torch.rand(K, C, 3, 3, device=dev, generator=g) - 0.5
    macs = float(torch.nn.functional.conv2d((x != 0).float().sum(1, keepdim=True), torch.ones(1,1,3,3,device=dev)).sum()) * K
    t = tm(lambda: sc.ecr_conv_batched(x, w, 1, fast=True, sync=False))
    out[name] = (round(t, 1), round(2 * macs / t / 1e6, 2))
print(json.dumps(out))
''' % ROOT
for cfg in sys.argv[1:] or ["1", "2", "3", "4", "5", "6"]:
    env = dict(os.environ, SCONV_TILED_CFG=cfg) if cfg[0].isdigit() else dict(os.environ, SCONV_KERNEL=cfg)
    r = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True)
    print("cfg", cfg, r.stdout.strip() or r.stderr[-500:], flush=True)
