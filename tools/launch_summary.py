"""Summarise an ncu launch list (tools/gpu_runs/gpu_r2_launches.sh) into
profiles/rNN/launches_latest.txt: the launches of the last bench step.

    python tools/launch_summary.py gpurun_out/launches.csv > profiles/r02/launches_latest.txt

The list holds warmup + timed steps of our kernels only; one step of the
VGG-19 bench is 32 launches (16 layers x filter transpose + conv kernel), so
the last 32 rows are the timed step.
"""
import csv
import sys

PER_STEP = 32


def main(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    ix = {k: i for i, k in enumerate(rows[0])}
    seq = [(r[ix["Kernel Name"]], float(r[ix["Metric Value"]].replace(",", "")))
           for r in rows[1:] if r[ix["Metric Name"]] == "gpu__time_duration.sum"]
    last = seq[-PER_STEP:]
    tot = sum(t for _, t in last) / 1e3
    print("# ncu launch list, one bench step (the last of warmup 3 + 1 timed), our kernels only")
    print("# ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised: compare shares)")
    print(f"# step total {tot:.1f} us over {len(last)} launches")
    for name, t in last:
        short = name.replace("sconv_cu::", "")
        print(f"{t / 1e3:9.1f} us {100 * t / 1e3 / tot:5.1f}%  {short}")


if __name__ == "__main__":
    main(sys.argv[1])
