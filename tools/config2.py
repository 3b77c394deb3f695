"""BASELINE config 2: the AlexNet / GoogLeNet / LeNet single layers of the
paper's Table, ECR conv on the B200 vs cuDNN, batch 64.

Spatial size and sparsity are the paper's; channel counts and kernel sizes
are not in the paper and come from the canonical model definitions
(LeNet-5 conv2; CaffeNet/AlexNet conv3, conv4; GoogLeNet inception 4a/4e/5a/5b
branches: .1 = 1x1 branch, .2 = 3x3 branch after its reduce, .3 = 5x5 branch
after its reduce; "4a.7" at 7x7 is taken as 4a's 1x1 pool projection).
Valid convolution on the stated map size, as the reference computes it.
Parity: EXACT output of image 0 vs the C oracle (bitwise); timing: CUDA
events, FAST arithmetic.  Prints one JSON line per layer.
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1909_09927_b200 as sc  # noqa: E402
from oracle.oracle import c_oracle  # noqa: E402

# name, C, K, k, size, sparsity
LAYERS = [
    ("LeNet.conv2", 20, 50, 5, 11, 0.95),
    ("AlexNetC.conv3", 256, 384, 3, 6, 0.9),
    ("AlexNetI.conv4", 384, 384, 3, 5, 0.9),
    ("GoogLeNet.inception4a.1", 480, 192, 1, 14, 0.9),
    ("GoogLeNet.inception4a.2", 96, 208, 3, 14, 0.9),
    ("GoogLeNet.inception4e.3", 32, 128, 5, 14, 0.9),
    ("GoogLeNet.inception5a.1", 832, 256, 1, 7, 0.95),
    ("GoogLeNet.inception5a.2", 160, 320, 3, 7, 0.9),
    ("GoogLeNet.inception5b.3", 48, 128, 5, 7, 0.95),
    ("GoogLeNet.inception4a.7", 480, 64, 1, 7, 0.95),
]
N = int(os.environ.get("N", 64))


def main():
    torch.backends.cudnn.allow_tf32 = False
    torch.backends.cudnn.benchmark = True
    dev = torch.device("cuda:0")
    orc = c_oracle()
    only = [o for o in os.environ.get("ONLY", "").split(",") if o]
    for name, C, K, k, size, s in LAYERS:
        if only and name not in only:
            continue
        x = np.stack([orc.generate(size, size, C, s, 7_000_000 + n) for n in range(N)])
        w = np.stack([orc.generate(k, k, C, 0.0, 8_000_000 + j) for j in range(K)]) - np.float32(0.5)
        ref, _ = orc.ecr_conv(x[:1], w, 1)
        y = sc.ecr_conv_batched(x[:1], w, 1)
        exact = bool(np.array_equal(y.view(np.uint32), ref.view(np.uint32)))
        xt, wt = torch.from_numpy(x).to(dev), torch.from_numpy(w).to(dev)
        plan = sc.launch_plan(N, C, size, size, K, k, k, 1)

        def tm(fn, reps=20):
            for _ in range(3):
                fn()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record()
            for _ in range(reps):
                fn()
            e1.record()
            torch.cuda.synchronize()
            return e0.elapsed_time(e1) / reps * 1e3
        ours = tm(lambda: sc.ecr_conv_batched(xt, wt, 1, fast=True, sync=False))
        cud = tm(lambda: torch.nn.functional.conv2d(xt, wt))
        row = {"layer": name, "C": C, "K": K, "k": k, "size": size, "sparsity": s,
               "N": N, "kernel": plan["kernel"], "exact_bitwise_vs_oracle": exact,
               "ours_us": round(ours, 2), "cudnn_us": round(cud, 2),
               "speedup_vs_cudnn": round(cud / ours, 3)}
        # KIDS=A,E,N,...: also time forced configs (dev sweep)
        for kid in filter(None, os.environ.get("KIDS", "").split(",")):
            try:
                row["us_" + kid] = round(tm(lambda: sc.ecr_conv_batched(
                    xt, wt, 1, fast=True, sync=False, kernel=kid)), 2)
            except Exception as e:  # config does not apply to this window
                row["us_" + kid] = str(e)[:24]
        print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
