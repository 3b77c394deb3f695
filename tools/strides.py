"""Paper stride experiments: VGG-19 layers with stride 2 and
3, ECR (FAST) on the B200 vs cuDNN, batch 64, s = 0.7; EXACT parity of image 0
against the C oracle.  One JSON line per (layer, stride)."""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import paper_1909_09927_b200 as sc
from oracle.oracle import c_oracle
LAYERS = [("conv2_2", 128, 128, 112), ("conv3_2", 256, 256, 56), ("conv4_2", 512, 512, 28),
          ("conv5_2", 512, 512, 14)]
N = int(os.environ.get("N", 64))
torch.backends.cudnn.allow_tf32 = False
torch.backends.cudnn.benchmark = True
dev = torch.device("cuda:0")
orc = c_oracle()
def tm(fn, reps=10):
    for _ in range(3): fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3
for name, C, K, H in LAYERS:
    g = torch.Generator(device=dev); g.manual_seed(3)
    x = torch.rand(N, C, H + 2, H + 2, device=dev, generator=g)
    x = x * (torch.rand(x.shape, device=dev, generator=g) >= 0.7)
    w = torch.rand(K, C, 3, 3, device=dev, generator=g) - 0.5
    for s in (1, 2, 3):
        ref, _ = orc.ecr_conv(x[:1].cpu().numpy(), w[:8].cpu().numpy(), s)
        y = sc.ecr_conv_batched(x[:1], w[:8], s)
        exact = bool(np.array_equal(y.cpu().numpy().view(np.uint32), ref.view(np.uint32)))
        plan = sc.launch_plan(N, C, H + 2, H + 2, K, 3, 3, s)
        ours = tm(lambda: sc.ecr_conv_batched(x, w, s, fast=True, sync=False))
        cud = tm(lambda: torch.nn.functional.conv2d(x, w, stride=s))
        print(json.dumps({"layer": name, "stride": s, "kernel": plan["kernel"], "exact": exact,
                          "ours_us": round(ours, 1), "cudnn_us": round(cud, 1),
                          "speedup_vs_cudnn": round(cud / ours, 3)}), flush=True)
