"""Time layer B right after layer A on one stream (dev probe: does A's
epilogue traffic leak into B's time?)."""
import os, sys, json, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1909_09927_b200 as sc
from paper_1909_09927_b200.workloads import VGG19, vgg_filters, vgg_maps
dev = torch.device("cuda:0")
names = os.environ.get("PAIR", "conv1_1,conv1_2").split(",")
ls = [[v[0] for v in VGG19].index(n) for n in names]
xs = [torch.from_numpy(vgg_maps(l, range(64), 0.7)).to(dev) for l in ls]
ws = [torch.from_numpy(vgg_filters(l)).to(dev) for l in ls]
def run(i):
    l = ls[i]
    if VGG19[l][4]:
        return sc.pecr_conv_pool_batched(xs[i], ws[i], 1, sc.PoolConfig(2, 2, 2), fast=True, sync=False)
    return sc.ecr_conv_batched(xs[i], ws[i], 1, fast=True, sync=False)
for _ in range(2):
    run(0); run(1)
torch.cuda.synchronize()
res = {"A_then_B": [], "B_alone": [], "A_alone": []}
for _ in range(5):
    e = [torch.cuda.Event(True) for _ in range(3)]
    e[0].record(); run(0); e[1].record(); run(1); e[2].record(); torch.cuda.synchronize()
    res["A_then_B"].append((e[0].elapsed_time(e[1]) * 1e3, e[1].elapsed_time(e[2]) * 1e3))
    e = [torch.cuda.Event(True) for _ in range(2)]
    torch.cuda.synchronize(); e[0].record(); run(1); e[1].record(); torch.cuda.synchronize()
    res["B_alone"].append(e[0].elapsed_time(e[1]) * 1e3)
    torch.cuda.synchronize(); e[0].record(); run(0); e[1].record(); torch.cuda.synchronize()
    res["A_alone"].append(e[0].elapsed_time(e[1]) * 1e3)
print(json.dumps({"pair": names, "A_in_pair": statistics.median(a for a, b in res["A_then_B"]),
                  "B_in_pair": statistics.median(b for a, b in res["A_then_B"]),
                  "B_alone": statistics.median(res["B_alone"]), "A_alone": statistics.median(res["A_alone"])}))
