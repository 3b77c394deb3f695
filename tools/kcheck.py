"""Dev tool: per-layer correctness (vs float64 torch conv) and timing of a
forced kernel family/config.  Usage: SCONV_KERNEL=i1 python tools/kcheck.py"""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1909_09927_b200 as sc
N = int(os.environ.get("N", 64)); S = float(os.environ.get("S", 0.7))
LAYERS = [("conv1_2",64,64,224,1),("conv2_2",128,128,112,1),("conv3_2",256,256,56,0),
          ("conv4_2",512,512,28,0),("conv4_4",512,512,28,1),("conv5_1",512,512,14,0)]
sel = os.environ.get("LAYERS")
if sel: LAYERS = [l for l in LAYERS if l[0] in sel.split(",")]
dev = torch.device("cuda:0")
def tm(fn, reps=5):
    for _ in range(2): fn()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    torch.cuda.synchronize(); s.record()
    for _ in range(reps): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / reps * 1000
out = {"kernel": os.environ.get("SCONV_KERNEL", "default")}
for name, C, K, Ho, pool in LAYERS:
    g = torch.Generator(device=dev); g.manual_seed(1)
    x = torch.rand(N, C, Ho + 2, Ho + 2, device=dev, generator=g)
    x = x * (torch.rand(x.shape, device=dev, generator=g) >= S)
    w = torch.rand(K, C, 3, 3, device=dev, generator=g) - 0.5
    macs = float(torch.nn.functional.conv2d((x != 0).float().sum(1, keepdim=True), torch.ones(1,1,3,3,device=dev)).sum()) * K
    for p in ([0, 1] if pool else [0]):
        if p:
            fn = lambda: sc.pecr_conv_pool_batched(x, w, 1, sc.PoolConfig(2, 2, 2), fast=True, sync=False)
        else:
            fn = lambda: sc.ecr_conv_batched(x, w, 1, fast=True, sync=False)
        y = fn(); torch.cuda.synchronize()
        nc = min(N, 4)
        ref = torch.nn.functional.conv2d(x[:nc].double(), w.double())
        if p: ref = torch.nn.functional.max_pool2d(torch.relu(ref), 2)
        d = (y[:nc].double() - ref).abs()
        bad = int((d > 1e-5 + 1e-5 * ref.abs()).sum())
        t = tm(fn)
        out[name + ("_pecr" if p else "")] = dict(us=round(t, 1), tflops=round(2 * macs / t / 1e6, 2),
                                                   maxabs=float(d.max()), bad=bad)
print(json.dumps(out), flush=True)
