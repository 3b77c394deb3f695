"""Accuracy-matched dense baselines on the bench's inputs (dev probe):
cuDNN's fastest fp32 algorithms (TF32 off) reach their speed with Winograd /
FFT, 36x outside the parity bar; this times the dense alternatives that do not
change the arithmetic that much -- PyTorch's native conv (cuDNN disabled:
im2col + cuBLAS SGEMM, TF32 off) and an explicit unfold + matmul -- and reports
each one's error against float64 as a multiple of 1e-5 + 1e-5|ref|."""
import json, os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1909_09927_b200.workloads import VGG19, vgg_filters, vgg_maps
dev = torch.device("cuda:0")
torch.backends.cudnn.allow_tf32 = False
torch.backends.cuda.matmul.allow_tf32 = False
names = os.environ.get("LAYERS", "conv3_2,conv4_2,conv5_1").split(",")
N = int(os.environ.get("N", "64"))
def t(fn, reps=3):
    fn(); torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(True), torch.cuda.Event(True)
        a.record(); fn(); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b) * 1e3)
    return statistics.median(ts)
for name in names:
    l = [v[0] for v in VGG19].index(name)
    x = torch.from_numpy(vgg_maps(l, range(N), 0.7)).to(dev)
    w = torch.from_numpy(vgg_filters(l)).to(dev)
    ref = torch.nn.functional.conv2d(x[:2].double(), w.double())
    out = {"layer": name}
    for mode in ("cudnn", "native"):
        torch.backends.cudnn.enabled = mode == "cudnn"
        torch.backends.cudnn.benchmark = True
        f = lambda: torch.nn.functional.conv2d(x, w)
        out[mode + "_us"] = t(f)
        y = torch.nn.functional.conv2d(x[:2], w).double()
        out[mode + "_err_x_bar"] = float(((y - ref).abs() / (1e-5 + 1e-5 * ref.abs())).max())
    torch.backends.cudnn.enabled = True
    print(json.dumps(out), flush=True)
