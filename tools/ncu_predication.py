"""Per-opcode executed counts, predicated-on fraction and stall-sample share
from an ncu --set full report's SASS source page (read here, no GPU).

    python tools/ncu_predication.py gpurun_out/c42_0.7.ncu-rep

`pred-on` = predicated-on thread instructions / (32 x warp instructions):
for FFMA2 under a predicate it is the fraction doing useful work.
"""
import collections
import csv
import io
import subprocess
import sys


def main(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    ix = {h: i for i, h in enumerate(hdr)}
    tot = collections.defaultdict(lambda: [0, 0, 0])
    samples = 0
    stalls = collections.Counter()
    cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    for r in rows[2:]:
        src = r[ix["Source"]].strip()
        if not src:
            continue
        f = src.split()
        pred = f[0].startswith("@")
        op = (f[1] if pred else f[0]).split(".")[0].rstrip(";")
        k = op + ("(pred)" if pred else "")
        ie = int(r[ix["Instructions Executed"]] or 0)
        te = int(r[ix["Predicated-On Thread Instructions Executed"]] or 0)
        s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
        t = tot[k]
        t[0] += ie
        t[1] += te
        t[2] += s
        samples += s
        for c in cols:
            stalls[c] += int(r[ix[c]] or 0)
    print(f"{'opcode':14s} {'warp inst':>12s} {'pred-on':>8s} {'samples':>8s}")
    for k, t in sorted(tot.items(), key=lambda kv: -kv[1][0])[:18]:
        print(f"{k:14s} {t[0]:12d} {t[1] / max(1, 32 * t[0]):8.3f} {100 * t[2] / samples:7.1f}%")
    st = sum(stalls.values())
    print("stall reasons (all samples): " +
          " ".join(f"{k[6:]}={100 * v / st:.1f}%" for k, v in stalls.most_common(8)))


if __name__ == "__main__":
    main(sys.argv[1])
