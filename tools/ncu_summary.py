"""Summarise an ncu --set full report (read here, no GPU): headline metrics,
instruction mix and not-issued stall reasons of the profiled kernel.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep > profiles/rNN/x.txt
"""
import collections
import csv
import io
import subprocess
import sys

KEYS = ["Duration", "Elapsed Cycles", "SM Frequency", "DRAM Throughput", "Compute (SM) Throughput",
        "Executed Ipc Active", "Issue Slots Busy", "Issued Warp Per Scheduler", "No Eligible",
        "Active Warps Per Scheduler", "Eligible Warps Per Scheduler",
        "Warp Cycles Per Issued Instruction", "Executed Instructions", "Registers Per Thread",
        "Dynamic Shared Memory Per Block", "Grid Size", "Block Size", "Achieved Occupancy",
        "Theoretical Occupancy", "L2 Hit Rate", "Memory Throughput"]


def ncu(rep, *args):
    return subprocess.run(["ncu", "-i", rep, *args, "--csv"], capture_output=True, text=True).stdout


def main(rep):
    det = list(csv.reader(io.StringIO(ncu(rep, "--page", "details"))))
    hdr = det[0]
    ik = hdr.index("Kernel Name")
    iname, iunit, ival = hdr.index("Metric Name"), hdr.index("Metric Unit"), hdr.index("Metric Value")
    print("kernel:", det[1][ik])
    seen = set()
    for r in det[1:]:
        if r[iname] in KEYS and r[iname] not in seen:
            seen.add(r[iname])
            print(f"  {r[iname]:40s} {r[ival]:>16s} {r[iunit]}")
    raw = list(csv.reader(io.StringIO(ncu(rep, "--page", "raw"))))
    h, units, vals = raw[0], raw[1], raw[2]
    for m in ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
              "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
              "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
              "smsp__inst_executed.sum"):
        if m in h:
            i = h.index(m)
            print(f"  {m:60s} {vals[i]:>16s} {units[i]}")
    src = list(csv.reader(io.StringIO(ncu(rep, "--page", "source", "--print-source", "sass"))))
    sh, data = src[1], src[2:]
    ie = sh.index("Instructions Executed")
    isamp = sh.index("Warp Stall Sampling (All Samples)")
    mix, samp = collections.Counter(), collections.Counter()
    for r in data:
        op = r[1].strip().split()
        if not op:
            continue
        o = op[1] if op[0].startswith("@") else op[0]
        o = o.split(".")[0]
        mix[o] += int(r[ie] or 0)
        samp[o] += int(r[isamp] or 0)
    T, S = sum(mix.values()), max(1, sum(samp.values()))
    print("instruction mix (executed, share, share of stall samples):")
    for o, n in mix.most_common(14):
        print(f"  {o:10s} {n:14d} {100 * n / T:5.1f}%  {100 * samp[o] / S:5.1f}%")
    cols = [i for i, x in enumerate(sh) if x.startswith("stall_") and "Not Issued" in x]
    tot = {sh[i]: sum(int(r[i] or 0) for r in data) for i in cols}
    S = max(1, sum(tot.values()))
    print("not-issued stall reasons:")
    for k, v in sorted(tot.items(), key=lambda x: -x[1])[:10]:
        print(f"  {k:40s} {100 * v / S:5.1f}%")


if __name__ == "__main__":
    main(sys.argv[1])
