"""Summarise an ncu launch list (tools/gpu_runs/gpu_r2_launches.sh) into
profiles/rNN/launches_latest.txt: the launches of the last bench step.

    python tools/launch_summary.py gpurun_out/launches.csv > profiles/r02/launches_latest.txt

The list holds warmup + timed steps of our kernels only; a step starts with
conv1_1 (filter transpose + the small-C kernel) and runs 2-4 launches per
layer (transpose, conv kernel; the 3x3 layers with a row-prefetch gate add
ws_density_gate_kernel and the instantiation that exits at once), so the
timed step is everything from the last conv1_1 transpose on.
"""
import csv
import sys


def main(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    ix = {k: i for i, k in enumerate(rows[0])}
    seq = [(r[ix["Kernel Name"]], float(r[ix["Metric Value"]].replace(",", "")))
           for r in rows[1:] if r[ix["Metric Name"]] == "gpu__time_duration.sum"]
    first = max(i for i, (n, _) in enumerate(seq) if "smallc" in n)
    if first > 0 and "transpose" in seq[first - 1][0]:
        first -= 1
    last = seq[first:]
    tot = sum(t for _, t in last) / 1e3
    print("# ncu launch list, one bench step (the last of warmup 3 + 1 timed), our kernels only")
    print("# ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised: compare shares)")
    print(f"# step total {tot:.1f} us over {len(last)} launches")
    for name, t in last:
        short = name.replace("sconv_cu::", "")
        print(f"{t / 1e3:9.1f} us {100 * t / 1e3 / tot:5.1f}%  {short}")


if __name__ == "__main__":
    main(sys.argv[1])
