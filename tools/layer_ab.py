"""A/B timing of single VGG-19 layers on the bench's own inputs (dev tool).

    LAYERS=conv1_1,conv4_2 S=0.7 python tools/layer_ab.py [ENV=VAL ...]

Each positional ENV=VAL group is one variant (comma-separated assignments,
e.g. SCONV_NO_SC2=1); the variant runs in a fresh subprocess so env-read
switches take effect.  Prints one JSON line per (variant, layer): CUDA-event
median of 5 launches after 2 warm-ups, device-resident inputs, plus a
bit-equality check of FAST output against variant 0 (same order => same bits).
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def child():
    sys.path.insert(0, ROOT)
    import numpy as np
    import torch
    import paper_1909_09927_b200 as sc
    from paper_1909_09927_b200.workloads import VGG19, vgg_filters, vgg_maps
    names = os.environ.get("LAYERS", "conv1_1").split(",")
    s = float(os.environ.get("S", "0.7"))
    n = int(os.environ.get("N", "64"))
    pecr_env = os.environ.get("PECR", "auto")
    fast = os.environ.get("EXACT", "0") != "1"  # EXACT=1: time the bit-exact mode
    dev = torch.device("cuda:0")
    out = {}
    for name in names:
        l = [v[0] for v in VGG19].index(name)
        _, C, K, H, pooled = VGG19[l]
        x = torch.from_numpy(vgg_maps(l, range(n), s)).to(dev)
        w = torch.from_numpy(vgg_filters(l)).to(dev)
        pecr = pooled if pecr_env == "auto" else pecr_env == "1"
        if pecr:
            fn = lambda: sc.pecr_conv_pool_batched(x, w, 1, sc.PoolConfig(2, 2, 2), fast=fast, sync=False)
        else:
            fn = lambda: sc.ecr_conv_batched(x, w, 1, fast=fast, sync=False)
        for _ in range(2):
            y = fn()
        ts = []
        for _ in range(5):
            a, b = torch.cuda.Event(True), torch.cuda.Event(True)
            torch.cuda.synchronize()
            a.record()
            y = fn()
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b) * 1000)
        ts.sort()
        nnz = (x != 0).float().sum(1, keepdim=True)
        box = torch.nn.functional.conv2d(nnz, torch.ones(1, 1, 3, 3, device=dev))
        flop = 2.0 * float(box.sum()) * K
        h = int(torch.from_numpy(np.frombuffer(y.cpu().numpy().tobytes(), dtype=np.uint8)).sum())
        out[name] = dict(us=ts[2], us_min=ts[0], tflops=flop / ts[2] / 1e6, pecr=pecr, bytesum=h)
    print("RESULT " + json.dumps(out), flush=True)


def main():
    variants = sys.argv[1:] or [""]
    base = None
    for v in variants:
        env = dict(os.environ)
        for kv in filter(None, v.split(",")):
            k, val = kv.split("=", 1)
            env[k] = val
        env["LAYER_AB_CHILD"] = "1"
        r = subprocess.run([sys.executable, __file__], env=env, capture_output=True, text=True)
        line = [x for x in r.stdout.splitlines() if x.startswith("RESULT ")]
        if not line:
            print(json.dumps({"variant": v, "error": (r.stdout + r.stderr)[-1500:]}), flush=True)
            continue
        res = json.loads(line[0][7:])
        if base is None:
            base = res
        for name, d in res.items():
            d["same_as_first"] = d["bytesum"] == base.get(name, {}).get("bytesum")
            print(json.dumps({"variant": v, "layer": name, **d}), flush=True)


if __name__ == "__main__":
    child() if os.environ.get("LAYER_AB_CHILD") else main()
