"""Refresh DESIGN.md section 8's measured numbers from a bench JSON line
(dev tool: python tools/refresh_design_status.py gpurun_out/bench.json)."""
import json
import re
import sys

d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
p = "DESIGN.md"
s = open(p).read()
L = d["layers"]
cu = d["cudnn"]["layers_us"]
s = re.sub(r"takes \*\*[\d.]+ ms = \d+ µs/layer\*\* \(round 1: 26.75 ms\),\n[\d.]+% of the FP32",
           f"takes **{d['ms_per_step']:.2f} ms = {d['value']:.0f} µs/layer** (round 1: 26.75 ms),\n"
           f"{d['roofline']['step_average']['frac'] * 100:.1f}% of the FP32", s)
s = re.sub(r"\(conv1_2 PECR\) [\d.]+ TFLOP/s = [\d.]+%, its DRAM traffic \d+ MB",
           f"(conv1_2 PECR) {d['roofline']['achieved']:.1f} TFLOP/s = {d['roofline']['frac'] * 100:.1f}%, "
           f"its DRAM traffic {d['roofline']['traffic'] / 1e6:.0f} MB", s)
s = re.sub(r"\*\*[\d.]+ ms per step\*\* on this box", f"**{d['e2e']['ms_per_step']:.1f} ms per step** on this box", s)
s = re.sub(r"dense ingest [\d.]+ ms\)", f"dense ingest {d['e2e']['dense']['ms_per_step']:.1f} ms)", s)
cb = d["cpu_baseline"]
s = re.sub(r"`oracle/_ref`\): \d+ s per layer extrapolated \(`workers = 1`: \d+ s; the\n×K×64 extrapolation checked "
           r"against a full-K conv5_1 run: ratio [\d.]+\)",
           f"`oracle/_ref`): {cb['value'] / 1e6:.0f} s per layer extrapolated (`workers = 1`: "
           f"{cb['workers_1']['value'] / 1e6:.0f} s; the\n×K×64 extrapolation checked against a full-K conv5_1 run: "
           f"ratio {cb['extrapolation_check']['ratio']:.2f})", s)
s = re.sub(r"[\d.]+ ms \([\d.]+×\)\. End to end",
           f"{d['cudnn']['ms_per_step']:.1f} ms ({d['cudnn']['speedup_ours_vs_cudnn']:.2f}×). End to end", s)
names = {"conv1_1": "3→64 @224", "conv1_2": "64→64 @224", "conv2_1": "64→128 @112", "conv2_2": "128→128 @112",
         "conv3_1": "128→256 @56", "conv3_2": "256→256 @56", "conv3_3": "256→256 @56", "conv3_4": "256→256 @56",
         "conv4_1": "256→512 @28", "conv4_2": "512→512 @28", "conv4_3": "512→512 @28", "conv4_4": "512→512 @28",
         "conv5_1": "512→512 @14", "conv5_2": "512→512 @14", "conv5_3": "512→512 @14", "conv5_4": "512→512 @14"}
rows = []
for k, v in L.items():
    kind = "PECR" if "PECR" in v["kernel"] else "ECR"
    extra = (f" (HBM-bound: {v['hbm_gbs'] / 1e3:.2f} TB/s = {v['hbm_frac'] * 100:.0f}% of HBM)"
             if k == "conv1_1" else "")
    rows.append(f"| {k} ({kind}) | {names[k]} | {v['us']:.0f} | {v['useful_tflops']:.1f}{extra} | "
                f"{v['fp32_frac'] * 100:.0f}% | {cu[k]:.0f} | {cu[k] / v['us']:.2f} |")
hdr = "| layer | C→K @H | µs | useful TFLOP/s | of FP32 peak | cuDNN µs | cuDNN / ours |"
i = s.index(hdr)
j = s.index("\n\nSparsity sweep", i)
s = s[:i] + hdr + "\n|---|---|---|---|---|---|---|\n" + "\n".join(rows) + s[j:]
sw = d["sweep"]["by_sparsity"]
swl = " ".join(f"s = {kk}: {vv['ms_per_step']:.1f} ms vs cuDNN {vv['cudnn_ms_per_step']:.1f} ms "
               f"({vv['speedup_vs_cudnn']:.2f}×, {vv['layers_won_vs_cudnn']} layers won);" for kk, vv in sw.items())
lead = "Sparsity sweep (reference-generator inputs, `bench.py` `sweep`): "
i = s.index(lead)
j = s.index(" from s ≈ 0.9", i)
s = s[:i] + lead + swl + s[j:]
s = re.sub(r"layer and is at \d+% there", f"layer and is at {L['conv1_1']['hbm_frac'] * 100:.0f}% there", s)
s = re.sub(r"holds on \d+\nof 16 at s = 0.7", f"holds on {d['cudnn']['layers_won']}\nof 16 at s = 0.7", s)
open(p, "w").write(s)
print("ok", d["ms_per_step"])
