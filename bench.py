"""bench.py -- VGG-19 ECR conv / PECR conv+pool on B200 (the BASELINE.json metric).

One step = the 16 VGG-19 conv layers at batch 64 (per GPU), sparsity 0.7,
valid 3x3 stride-1 convolution on pre-padded (H+2)x(W+2) inputs:
the 11 conv-only layers through the fused ECR kernel and the 5 layers
followed by 2x2/2 max-pooling through the fused PECR conv+ReLU+pool kernel
(the layer assignment of the reference's forward(net, Method::kPecr),
src/pipeline.cpp:234-264).  Every layer gets its own synthetic input, made
by the reference's generator (bit-identical sconv_generate):
    map  n of layer l:  generate(H+2, W+2, C, 0.7, 1e6*(l+1) + n)
    filt k of layer l:  generate(3, 3, C, 0, 1e6*(l+1) + 5e5 + k) - 0.5
Inputs are device resident when `value` is timed; `e2e` runs the same step
through the C ABI with pinned host buffers (H2D + kernel + D2H per layer).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
                    [--sparsity S] [--exact] [--sweep] [--no-cudnn]

Rank 0 prints ONE JSON line.  `--impl reference` times the reference's own
CPU implementation (oracle/_ref, built from /root/reference/proj/src) on the
host cores on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# VGG-19 conv layers: (name, C, K, H_out, pooled?)  -- SURVEY.md 8(d)
VGG19 = [
    ("conv1_1", 3, 64, 224, False), ("conv1_2", 64, 64, 224, True),
    ("conv2_1", 64, 128, 112, False), ("conv2_2", 128, 128, 112, True),
    ("conv3_1", 128, 256, 56, False), ("conv3_2", 256, 256, 56, False),
    ("conv3_3", 256, 256, 56, False), ("conv3_4", 256, 256, 56, True),
    ("conv4_1", 256, 512, 28, False), ("conv4_2", 512, 512, 28, False),
    ("conv4_3", 512, 512, 28, False), ("conv4_4", 512, 512, 28, True),
    ("conv5_1", 512, 512, 14, False), ("conv5_2", 512, 512, 14, False),
    ("conv5_3", 512, 512, 14, False), ("conv5_4", 512, 512, 14, True),
]
BATCH = 64
METRIC = "ECR conv / PECR conv+pool µs per VGG-19 layer; achieved GB/s vs HBM peak"
UNIT = "us/layer"


def map_seed(l, n):
    return 1_000_000 * (l + 1) + n


def filt_seed(l, k):
    return 1_000_000 * (l + 1) + 500_000 + k


def peaks():
    p = {"hbm_gbs": 6556.5, "sm_max_mhz": 1965.0, "src": "fallback"}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            m = json.load(f)
        p.update(hbm_gbs=m["hbm_gbs"], sm_max_mhz=m.get("sm_max_mhz", 1965.0), src="measured")
    except Exception:
        pass
    return p


# ---------------------------------------------------------------------------
# clocks sampled during the timed region
# ---------------------------------------------------------------------------
class ClockSampler:
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([v.strip() for v in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if len(r) > 3 + i and r[3 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


# ---------------------------------------------------------------------------
# reference / CPU arm
# ---------------------------------------------------------------------------
def cpu_lib():
    """The reference CPU implementation: oracle/_ref (unmodified reference
    sources) when built, else the C restatement (port)."""
    from oracle import oracle
    r = oracle.ref_lib()
    if r is not None:
        return r, "reference"
    return oracle.c_oracle(), "port"


def cpu_sample(lib, kind, step: int, filters_per_layer: int = 1):
    """Time ecr_convert+ecr_spmv_conv (or pecr_convert+pecr_conv_pool) for 1
    image x `filters_per_layer` filters per VGG-19 layer, as cmd_sweep times
    it (tools/sparseconv_main.cpp:365-368).  Returns per-layer seconds per
    (image, filter) and the total sample seconds."""
    import numpy as np
    workers = os.cpu_count() or 1
    per = {}
    total = 0.0
    for l, (name, C, K, H, pooled) in enumerate(VGG19):
        x = lib.generate(H + 2, H + 2, C, 0.7, map_seed(l, step % BATCH))[None]
        ks = [(step * filters_per_layer + j) % K for j in range(filters_per_layer)]
        w = np.stack([lib.generate(3, 3, C, 0.0, filt_seed(l, k)) for k in ks]) - np.float32(0.5)
        t0 = time.perf_counter()
        if kind == "reference":
            if pooled:
                lib.pecr_conv(x, w, 1, 2, 2, 2, 0, workers=workers)
            else:
                lib.ecr_conv(x, w, 1, workers=workers)
        else:
            if pooled:
                lib.pecr_conv(x, w, 1, 2, 2, 2, 0)
            else:
                lib.ecr_conv(x, w, 1)
        dt = time.perf_counter() - t0
        per[name] = dt / len(ks)
        total += dt
    return per, total


def run_reference(args):
    rank = int(os.environ.get("RANK", 0))
    if rank != 0:
        return 0
    lib, kind = cpu_lib()
    cores = (os.cpu_count() or 1) if kind == "reference" else 1
    for s in range(args.warmup):
        cpu_sample(lib, kind, 1000 + s)
    times = []
    per_layer_acc = {n: 0.0 for n, *_ in VGG19}
    for s in range(args.steps):
        per, _ = cpu_sample(lib, kind, s, filters_per_layer=4)
        # extrapolate the sample to the full layer: x K filters x 64 images
        step_us = 0.0
        for name, C, K, H, pooled in VGG19:
            us = per[name] * K * BATCH * 1e6
            per_layer_acc[name] += us
            step_us += us
        times.append(step_us)
    step_us = statistics.mean(times)
    value = step_us / len(VGG19)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": step_us / 1e3, "higher_is_better": False, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic (sconv::generate)",
        "config": {"workload": "VGG-19 16 conv layers (11 ECR + 5 PECR conv+pool), batch 64, "
                               "sparsity 0.7", "global_batch": BATCH, "sparsity": 0.7,
                   "sample": "1 image x 4 filters per layer per step, extrapolated x K x 64"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": kind,
                         "sample": "1 image x 4 filters per layer per step (extrapolated x K x 64)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "layers_us": {n: v / args.steps for n, v in per_layer_acc.items()},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--sparsity", type=float, default=0.7)
    ap.add_argument("--exact", action="store_true", help="EXACT (bit-exact) arithmetic")
    ap.add_argument("--no-cudnn", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--sweep", action="store_true", help="also sweep sparsity (side file)")
    ap.add_argument("--no-forward", action="store_true", help="skip the multi-layer forward leg")
    ap.add_argument("--no-check", action="store_true",
                    help="skip the accuracy spot check (profiling runs: keeps cuDNN out of the launch list)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)

    import numpy as np
    import torch
    import torch.distributed as dist
    import paper_1909_09927_b200 as sc

    world = int(os.environ.get("WORLD_SIZE", 1))
    rank = int(os.environ.get("RANK", 0))
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    torch.backends.cudnn.allow_tf32 = False
    torch.backends.cuda.matmul.allow_tf32 = False
    torch.backends.cudnn.benchmark = True
    fast = not args.exact
    sp = args.sparsity

    # ---- inputs: this rank's 64 images per layer (weak scaling) ---------
    t_gen = time.time()
    host_x, host_w, dev_x, dev_w, outs, macs = [], [], [], [], [], []
    for l, (name, C, K, H, pooled) in enumerate(VGG19):
        seeds = [map_seed(l, rank * BATCH + n) for n in range(BATCH)]
        hx = torch.empty((BATCH, C, H + 2, H + 2), dtype=torch.float32, pin_memory=True)
        sc.generate_batch(seeds, H + 2, H + 2, C, sp, out=hx.numpy())
        hw = torch.empty((K, C, 3, 3), dtype=torch.float32, pin_memory=True)
        sc.generate_batch([filt_seed(l, k) for k in range(K)], 3, 3, C, 0.0, out=hw.numpy())
        hw -= 0.5
        host_x.append(hx)
        host_w.append(hw)
        dx = hx.to(dev, non_blocking=True)
        dw = hw.to(dev, non_blocking=True)
        dev_x.append(dx)
        dev_w.append(dw)
        oh = H // 2 if pooled else H
        outs.append(torch.empty((BATCH, K, oh, oh), dtype=torch.float32, device=dev))
        # useful MACs = K * sum over images/windows of window nnz (== OpCount.multiplications)
        nz = (dx != 0).to(torch.float32).sum(1, keepdim=True)
        win = torch.nn.functional.conv2d(nz, torch.ones(1, 1, 3, 3, device=dev))
        macs.append(float(win.sum().item()) * K)
    torch.cuda.synchronize()
    t_gen = time.time() - t_gen

    ctx = sc.context(local)
    stream = torch.cuda.current_stream(dev)
    pool_cfg = sc.PoolConfig(2, 2, 2, sc.PoolMode.kMax)

    def layer(l):
        name, C, K, H, pooled = VGG19[l]
        if pooled:
            sc.pecr_conv_pool_batched(dev_x[l], dev_w[l], 1, pool_cfg, fast=fast, out=outs[l],
                                      sync=False)
        else:
            sc.ecr_conv_batched(dev_x[l], dev_w[l], 1, fast=fast, out=outs[l], sync=False)

    # Accuracy spot check at full size (images 0-1 of every layer) against a
    # float64 convolution: the north-star bar |d| <= 1e-5 + 1e-5|ref| as a
    # ratio (<= 1 passes) for our output and for cuDNN fp32 (TF32 off).  The
    # reference's own fp32 sum also deviates from float64 (its order differs),
    # so the ratio of the oracle itself sits near 1; tests/ pin the oracle.
    max_rel = 0.0
    acc_ratio = {"ours_vs_reference": 0.0, "cudnn_vs_reference": 0.0, "ours_vs_f64": 0.0,
                 "cudnn_vs_f64": 0.0}
    for l, (name, C, K, H, pooled) in enumerate(VGG19):
        layer(l)
        if args.no_check:
            continue
        x2 = dev_x[l][:2]
        # the reference's own fp32 result: EXACT mode is bit-identical to it
        # (tests/test_gpu_parity.py, full VGG shapes included)
        if pooled:
            refx = sc.pecr_conv_pool_batched(x2, dev_w[l], 1, pool_cfg, fast=False)
        else:
            refx = sc.ecr_conv_batched(x2, dev_w[l], 1, fast=False)
        ref64 = torch.nn.functional.conv2d(x2.double(), dev_w[l].double())
        ref32 = torch.nn.functional.conv2d(x2, dev_w[l])
        if pooled:
            ref64 = torch.nn.functional.max_pool2d(torch.relu(ref64), 2)
            ref32 = torch.nn.functional.max_pool2d(torch.relu(ref32), 2)
        got, cud, rx = outs[l][:2].double(), ref32.double(), refx.double()
        for tag, ref in (("reference", rx), ("f64", ref64)):
            tol = 1e-5 + 1e-5 * ref.abs()
            acc_ratio["ours_vs_" + tag] = max(acc_ratio["ours_vs_" + tag],
                                              ((got - ref).abs() / tol).max().item())
            acc_ratio["cudnn_vs_" + tag] = max(acc_ratio["cudnn_vs_" + tag],
                                               ((cud - ref).abs() / tol).max().item())
        err = ((got - cud).abs() / (1e-3 + cud.abs())).max().item()
        max_rel = max(max_rel, err)
    torch.cuda.synchronize()

    for _ in range(args.warmup):
        for l in range(len(VGG19)):
            layer(l)
    torch.cuda.synchronize()

    # ---- timed region: K steps, events per layer --------------------------
    nl = len(VGG19)
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(nl + 1)] for _ in range(args.steps)]
    launches0 = ctx.launches
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for s in range(args.steps):
            ev[s][0].record(stream)
            for l in range(nl):
                layer(l)
                ev[s][l + 1].record(stream)
        torch.cuda.synchronize()
    launches = ctx.launches - launches0
    if world > 1:
        dist.barrier()
    step_ms = [ev[s][0].elapsed_time(ev[s][nl]) for s in range(args.steps)]
    layer_ms = [statistics.mean(ev[s][l].elapsed_time(ev[s][l + 1]) for s in range(args.steps))
                for l in range(nl)]
    total_ms = sum(step_ms)
    if world > 1:
        t = torch.tensor([total_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = t.item()
    ms_per_step = total_ms / args.steps

    # ---- roofline of the dominant kernel (the fused ECR/PECR kernel) ------
    pk = peaks()
    flops = [2 * m for m in macs]
    in_bytes = [x.numel() * 4 for x in dev_x]
    w_bytes = [w.numel() * 4 for w in dev_w]
    out_bytes = [o.numel() * 4 for o in outs]
    alg_bytes = [a + b + c for a, b, c in zip(in_bytes, w_bytes, out_bytes)]
    clocks = clk.summary()
    fp32_peak = 148 * 128 * 2 * pk["sm_max_mhz"] * 1e6 / 1e12  # TFLOP/s at max SM clock
    achieved_tf = sum(flops) / (sum(layer_ms) * 1e-3) / 1e12
    achieved_gbs = sum(alg_bytes) / (sum(layer_ms) * 1e-3) / 1e9
    dom = max(range(nl), key=lambda l: layer_ms[l])
    traffic = None  # DRAM bytes of the dominant layer's launch, from the committed ncu capture
    try:
        with open(os.path.join(ROOT, "profiles", "r01", "traffic.json")) as f:
            t = json.load(f).get(VGG19[dom][0])
        if t:
            traffic = t["dram_read_bytes"] + t["dram_write_bytes"]
    except Exception:
        pass

    # ---- cuDNN dense comparison (same inputs, same GPU) -------------------
    cudnn = {}
    if not args.no_cudnn:
        def dense(l):
            name, C, K, H, pooled = VGG19[l]
            y = torch.nn.functional.conv2d(dev_x[l], dev_w[l])
            if pooled:
                y = torch.nn.functional.max_pool2d(torch.relu(y), 2)
            return y
        for l in range(nl):
            for _ in range(2):
                dense(l)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        per = []
        for l in range(nl):  # best of 3 trials of 3 launches: cuDNN at its fastest
            best = None
            for _ in range(3):
                e0.record(stream)
                for _ in range(3):
                    dense(l)
                e1.record(stream)
                torch.cuda.synchronize()
                t = e0.elapsed_time(e1) / 3
                best = t if best is None else min(best, t)
            per.append(best)
        cudnn = {"ms_per_step": sum(per), "us_per_layer": sum(per) * 1e3 / nl,
                 "layers_us": {VGG19[l][0]: per[l] * 1e3 for l in range(nl)},
                 "speedup_ours_vs_cudnn": sum(per) / ms_per_step,
                 "settings": "torch conv2d(padding=0)+relu+max_pool2d, fp32, TF32 off, "
                             "cudnn.benchmark=True, best of 3 trials per layer"}

    # ---- e2e through the C ABI with pinned host buffers --------------------
    e2e = None
    if not args.no_e2e:
        host_out = [torch.empty(o.shape, dtype=torch.float32, pin_memory=True) for o in outs]
        xs = [h.numpy() for h in host_x]
        ws = [h.numpy() for h in host_w]
        ys = [h.numpy() for h in host_out]

        def e2e_step():
            # one asynchronous C-ABI call per layer (host pointers: each call
            # owns a workspace and its H2D / compute / D2H ring, so layer l+1's
            # input copy overlaps layer l's compute and output copy), then one
            # synchronisation: every H2D and D2H byte is inside the step
            for l, (name, C, K, H, pooled) in enumerate(VGG19):
                if pooled:
                    sc.pecr_conv_pool_batched(xs[l], ws[l], 1, pool_cfg, fast=fast, out=ys[l],
                                              device=local, sync=False)
                else:
                    sc.ecr_conv_batched(xs[l], ws[l], 1, fast=fast, out=ys[l], device=local,
                                        sync=False)
            sc.synchronize(local)
        for _ in range(3):  # sizes the per-call workspaces and the memory pool
            e2e_step()
        if world > 1:
            dist.barrier()
        e2e_steps = max(1, min(args.steps, 5))
        e2e_each = []
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            t1 = time.perf_counter()
            e2e_step()
            e2e_each.append(round((time.perf_counter() - t1) * 1e3, 2))
        e2e_ms = (time.perf_counter() - t0) * 1e3 / e2e_steps
        if world > 1:
            t = torch.tensor([e2e_ms], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_ms = t.item()
        h2d = sum(in_bytes) + sum(w_bytes)
        d2h = sum(out_bytes)
        e2e = {"value": e2e_ms * 1e3 / nl / world, "unit": UNIT, "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "ms_per_step": e2e_ms, "ms_each_step": e2e_each,
               "path": "sconv_cu_ecr_conv / sconv_cu_pecr_conv_pool with pinned host pointers, "
                       "SCONV_F_ASYNC per layer + one sconv_cu_synchronize per step"}

    # ---- CPU reference sample on this host (rank 0 only, N=1 only) --------
    cpu = None
    if not args.no_cpu and rank == 0 and world == 1:
        try:
            lib, kind = cpu_lib()
            cpu_sample(lib, kind, 0)  # warm
            per, total = cpu_sample(lib, kind, 1, filters_per_layer=48)  # ~10 s of CPU work
            est_us = sum(per[n] * K * BATCH * 1e6 for n, C, K, H, p in VGG19)
            cpu = {"value": est_us / nl, "unit": UNIT,
                   "cores": (os.cpu_count() or 1) if kind == "reference" else 1, "kind": kind,
                   "sample": f"1 image x 48 filters per layer ({total:.1f} s), extrapolated x K x 64",
                   "speedup_ours_vs_cpu": (est_us / 1e3) / ms_per_step}
        except Exception as exc:  # the GPU number stands without it
            cpu = {"value": None, "error": str(exc)[:200]}

    if args.sweep and rank == 0:
        sweep_side_file(sc, torch, dev, fast)

    fwd = None if args.no_forward else forward_side(sc, torch, dev, fast, rank)

    value = ms_per_step * 1e3 / nl / world
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": False,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (sconv::generate, bit-identical to the reference generator)",
        "config": {
            "workload": "VGG-19 16 conv layers: 11 ECR conv + 5 PECR conv+ReLU+maxpool2x2, "
                        "batch 64 per GPU, sparsity %.2f, valid 3x3 s1 on pre-padded inputs" % sp,
            "global_batch": BATCH * world, "sparsity": sp, "parallelism": f"batch-shard x{world}",
            "arith": "FAST (FFMA, |d|<=1e-5+1e-5|ref|)" if fast else "EXACT (bit-exact)",
            "l2": "inputs larger than L2: 2.8 GB of inputs per step, every layer's input is "
                  "evicted by the other 15 layers' traffic before it is read again",
            "seeds": "map 1e6*(l+1)+n, filter 1e6*(l+1)+5e5+k, filters - 0.5",
        },
        "images_per_s": BATCH * world / (ms_per_step * 1e-3),
        "layers_us": {VGG19[l][0]: layer_ms[l] * 1e3 for l in range(nl)},
        "roofline": {
            "bound": "fp32", "achieved": achieved_tf, "peak": fp32_peak, "unit": "TFLOP/s",
            "frac": achieved_tf / fp32_peak, "traffic": traffic,
            "traffic_what": "dram__bytes_read+write of one launch of the dominant layer "
                            "(profiles/r01/traffic.json) vs its algorithmic bytes "
                            "dominant_layer_alg_bytes",
            "dominant_layer_alg_bytes": alg_bytes[dom],
            "what": "useful (nonzero) FLOPs of the fused ECR/PECR kernel over its event time; "
                    "peak = FP32 FFMA 148 SM x 128 x 2 x sm_max_mhz (not in MEASURED_PEAKS)",
            "hbm": {"achieved_gbs": achieved_gbs, "peak_gbs": pk["hbm_gbs"],
                    "frac": achieved_gbs / pk["hbm_gbs"], "peak_src": pk["src"],
                    "bytes": "compulsory: inputs + filters + outputs"},
            "dominant_layer": VGG19[dom][0],
            "dominant_layer_tflops": flops[dom] / (layer_ms[dom] * 1e-3) / 1e12,
        },
        "useful_gflop_per_step": sum(flops) / 1e9,
        "max_rel_err_vs_cudnn": max_rel,
        "accuracy": {k: round(v, 3) for k, v in acc_ratio.items()},
        "accuracy_what": "max over all 16 layers (images 0-1) of |out - ref| / (1e-5 + 1e-5|ref|)"
                         " with ref = the reference's fp32 result (our EXACT mode, bit-identical"
                         " to it) or a float64 convolution; <= 1 meets the north-star bar",
        "gpu_launches": launches,
        "clocks": clocks,
        "cudnn": cudnn or None,
        "e2e": e2e,
        "cpu_baseline": cpu,
        "forward": fwd,
        "setup_s": t_gen,
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


# VGG-19 on valid convolutions (the reference's forward() has no padding): a
# 460x460 input gives VGG-19's block structure (2-2-4-4-4 convs, 2x2/2 max
# pools after each block) and ends at 512 x 7 x 7.
FWD_IN = 460
FWD_BATCH = 16


def vgg19_valid_layers():
    chans = [(3, 64), (64, 64), (64, 128), (128, 128), (128, 256), (256, 256), (256, 256),
             (256, 256), (256, 512), (512, 512), (512, 512), (512, 512), (512, 512), (512, 512),
             (512, 512), (512, 512)]
    pooled = {1, 3, 7, 11, 15}
    return [(c, k, l in pooled) for l, (c, k) in enumerate(chans)]


def forward_side(sc, torch, dev, fast, rank):
    """forward(net, x, Method::kPecr) of pipeline.cpp:212-301 on the GPU
    (sconv_cu_forward): VGG-19 (valid convs) with ReLU, the 5 pooled layers
    fused (PECR), activations resident in HBM between layers.  Timed with CUDA
    events on the context stream, device-resident input and filters."""
    spec = vgg19_valid_layers()
    layers = []
    for l, (c, k, pooled) in enumerate(spec):
        hw = torch.empty((k, c, 3, 3), dtype=torch.float32)
        sc.generate_batch([2_000_000 * (l + 1) + j for j in range(k)], 3, 3, c, 0.0,
                          out=hw.numpy())
        hw -= 0.5
        # scale so activations stay O(1) through 16 layers (He-style)
        hw *= float((2.0 / (9 * c)) ** 0.5 / 0.29)
        layers.append({"filters": hw.to(dev), "stride": 1, "relu": True,
                       "pool": sc.PoolConfig(2, 2, 2) if pooled else None})
    hx = torch.empty((FWD_BATCH, 3, FWD_IN, FWD_IN), dtype=torch.float32)
    sc.generate_batch([3_000_000 + rank * FWD_BATCH + n for n in range(FWD_BATCH)], FWD_IN,
                      FWD_IN, 3, 0.7, out=hx.numpy())
    x = hx.to(dev)
    run = lambda: sc.forward_batched(x, layers, sc.Method.kPecr, fast=fast)
    y, _, _, fb = run()
    run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 3
    e0.record()
    for _ in range(reps):
        run()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    nz = float((y != 0).float().mean().item())
    # batch-1 latency, eager launches vs one CUDA-graph replay (SCONV_F_GRAPH)
    x1 = x[:1].contiguous()
    y1 = torch.empty((1,) + tuple(y.shape[1:]), dtype=torch.float32, device=dev)
    lat = {}
    for tag, graph in (("eager", False), ("graph", True)):
        f1 = lambda: sc.forward_batched(x1, layers, sc.Method.kPecr, fast=fast, graph=graph, out=y1)
        f1()
        f1()
        torch.cuda.synchronize()
        e0.record()
        for _ in range(10):
            f1()
        e1.record()
        torch.cuda.synchronize()
        lat[tag] = e0.elapsed_time(e1) / 10
    return {"network": "VGG-19 valid convs (16 conv + ReLU, 5 fused 2x2/2 max pools), input "
                       f"3x{FWD_IN}x{FWD_IN}, batch {FWD_BATCH} per GPU, input sparsity 0.7",
            "ms_per_batch": ms, "images_per_s": FWD_BATCH / (ms * 1e-3),
            "output_shape": list(y.shape), "pecr_fallback_layers": fb,
            "output_nonzero_frac": nz,
            "batch1_ms": lat,
            "path": "sconv_cu_forward (one call, device pointers)"}


def sweep_side_file(sc, torch, dev, fast):
    """Sparsity sweep per layer (ECR for all 16 layers, PECR for the pooled
    ones), written to profiles/sweep_latest.json (not the bench line)."""
    res = []
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for s in (0.5, 0.6, 0.7, 0.8, 0.9, 0.95):
        for l, (name, C, K, H, pooled) in enumerate(VGG19):
            g = torch.Generator(device=dev)
            g.manual_seed(l)
            x = torch.rand(BATCH, C, H + 2, H + 2, device=dev, generator=g)
            x = x * (torch.rand(x.shape, device=dev, generator=g) >= s)
            w = torch.rand(K, C, 3, 3, device=dev, generator=g) - 0.5
            macs = float(torch.nn.functional.conv2d((x != 0).float().sum(1, keepdim=True),
                                                    torch.ones(1, 1, 3, 3, device=dev)).sum()) * K
            row = {"sparsity": s, "layer": name}
            for tag, fn in (("ecr", lambda: sc.ecr_conv_batched(x, w, 1, fast=fast, sync=False)),
                            ("cudnn", lambda: torch.nn.functional.conv2d(x, w))):
                fn()
                ev0.record()
                for _ in range(3):
                    fn()
                ev1.record()
                torch.cuda.synchronize()
                row[tag + "_us"] = ev0.elapsed_time(ev1) / 3 * 1e3
            if pooled:
                pc = sc.PoolConfig(2, 2, 2)
                for tag, fn in (("pecr", lambda: sc.pecr_conv_pool_batched(x, w, 1, pc, fast=fast,
                                                                           sync=False)),
                                ("cudnn_pool", lambda: torch.nn.functional.max_pool2d(
                                    torch.relu(torch.nn.functional.conv2d(x, w)), 2))):
                    fn()
                    ev0.record()
                    for _ in range(3):
                        fn()
                    ev1.record()
                    torch.cuda.synchronize()
                    row[tag + "_us"] = ev0.elapsed_time(ev1) / 3 * 1e3
            row["useful_tflops"] = 2 * macs / (row["ecr_us"] * 1e-6) / 1e12
            res.append(row)
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    with open(os.path.join(ROOT, "profiles", "sweep_latest.json"), "w") as f:
        json.dump(res, f, indent=1)


if __name__ == "__main__":
    sys.exit(main())
