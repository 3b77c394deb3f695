"""Generate tests/golden/reference_vectors.json by running the UNMODIFIED
reference library (oracle/_ref/libsconv_ref.so, built by oracle/Makefile from
/root/reference/proj/src).  Run in the dev container, where the reference is
mounted:

    make -C oracle ref && python tests/golden/make_golden.py

The fixtures pin the C oracle (tests/test_oracle.py) and the GPU path
(tests/test_gpu_*.py) on machines where the reference is absent.  Inputs are
regenerated from seeds with sconv::generate, so only checksums, counters and
small arrays are stored.
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), "..", ".."))
sys.path.insert(0, ROOT)
from oracle.oracle import OracleError, RefLib  # noqa: E402

OUT = os.path.join(os.path.dirname(__file__), "reference_vectors.json")


def main() -> None:
    r = RefLib()
    g: dict = {"source": "oracle/_ref/libsconv_ref.so built from /root/reference/proj/src"}

    # Rng test vectors (test_dataset.cpp:43-48) and a few more seeds
    g["rng"] = {str(s): ["%016x" % v for v in r.rng(s, 5)] for s in (0, 1, 42, 20250801)}

    # generate(): checksums and exact zero counts
    gen = []
    for (h, w, c, s, seed) in [(32, 32, 1, 0.7, 42), (6, 6, 2, 1.0, 9), (6, 6, 2, 0.0, 9),
                               (17, 13, 2, 0.5, 31), (226, 226, 3, 0.7, 1000000),
                               (58, 58, 128, 0.7, 5000003), (16, 16, 512, 0.95, 7)]:
        m = r.generate(h, w, c, s, seed)
        gen.append(dict(h=h, w=w, c=c, s=s, seed=seed, checksum=r.checksum(m),
                        zeros=int((m == 0).sum())))
    g["generate"] = gen

    # fixtures F5 / K3 and their frozen answers
    f5, k3 = r.fixtures()
    dense, ops = r.dense_conv(f5, k3, 1)
    e = r.ecr_convert(f5, k3, 1)
    p = r.pecr_convert(f5, k3, 1, 2, 2, 1)
    pooled, pops = r.pecr_conv(f5[None], k3[None], 1, 2, 2, 1, 0)
    mean, _ = r.pecr_conv(f5[None], k3[None], 1, 2, 2, 1, 1)
    g["fixtures"] = dict(
        f5=f5.reshape(-1).tolist(), k3=k3.reshape(-1).tolist(),
        dense=dense.reshape(-1).tolist(), dense_ops=list(ops),
        ecr_ptr=e["ptr"].reshape(-1).tolist(), ecr_offsets=e["offsets"].reshape(-1).tolist(),
        ecr_f=e["f_data"].reshape(-1).tolist(), ecr_k=e["k_data"].reshape(-1).tolist(),
        pecr_count=p["count"].reshape(-1).tolist(), pecr_start=p["pack_start"].tolist(),
        pecr_data=p["data"].tolist(), pecr_index=p["index"].tolist(),
        pecr_max=pooled.reshape(-1).tolist(), pecr_ops=list(pops),
        pecr_mean=mean.reshape(-1).tolist())

    # Seeded KATs: w = generate(3,3,C,0,ws) - 0.5, pool 2x2 s2 max
    kats = []
    for (c, h, s, ms, ws) in [(3, 16, .7, 7, 8), (16, 34, .7, 101, 202), (64, 30, .9, 303, 404),
                              (512, 16, .7, 505, 606)]:
        x = r.generate(h, h, c, s, ms)
        w = r.generate(3, 3, c, 0.0, ws) - np.float32(0.5)
        y, eops = r.ecr_conv(x[None], w[None], 1)
        pc, pops = r.pecr_conv(x[None], w[None], 1, 2, 2, 2, 0)
        kats.append(dict(c=c, h=h, s=s, ms=ms, ws=ws, map=r.checksum(x), ecr=r.checksum(y),
                         pecr=r.checksum(pc), ecr_ops=list(eops), pecr_ops=list(pops)))
    g["kats"] = kats

    # pecr_pack_count cases (test_pecr.cpp:46-60)
    pcs = []
    for args in [(5, 3, 1, 2, 1), (3, 3, 1, 1, 1), (12, 3, 1, 2, 2), (12, 3, 1, 3, 2),
                 (6, 3, 2, 2, 1), (5, 3, 1, 7, 1), (5, 3, 0, 2, 1), (226, 3, 1, 2, 2),
                 (16, 3, 1, 2, 2), (9, 3, 2, 2, 1)]:
        try:
            pcs.append(dict(args=list(args), packs=r.pack_count(*args)))
        except OracleError as ex:
            pcs.append(dict(args=list(args), error=ex.kind))
    g["pack_count"] = pcs

    # plan() (test_exec.cpp:23-44)
    g["plan"] = [dict(args=[64, 64, 3, 3, 1, 1, 0, 0, 0, 1], out=list(r.plan(64, 64, 3, 3, 1, 1))),
                 dict(args=[5, 5, 3, 3, 1, 1, 1, 2, 2, 1],
                      out=list(r.plan(5, 5, 3, 3, 1, 1, 1, 2, 2, 1)))]

    # A seeded sweep in the style of acceptance_main.cpp:62-79: ECR format +
    # output + counters, PECR format + max/mean outputs where Eq. 3 tiles.
    sweep = []
    seeds = r.rng(20250801, 200)
    sp = [0.0, 0.5, 0.7, 0.9, 1.0]
    i = 0
    while len(sweep) < 40:
        a, b, cc, d, e_ = seeds[i:i + 5]
        i += 5
        size = 5 + a % 40
        k = 3 if b % 2 == 0 else 5
        if k > size:
            continue
        stride = 1 + cc % 3
        ch = 1 if d % 2 == 0 else 3
        s = sp[e_ % 5]
        ms, ws = (a ^ e_) & 0xFFFFFFFF, (b ^ d) & 0xFFFFFFFF
        x = r.generate(size, size, ch, s, ms)
        w = r.generate(k, k, ch, 0.0, ws)
        if len(sweep) % 2:
            w = w - np.float32(0.5)
        e = r.ecr_convert(x, w, stride)
        y, eops = r.ecr_conv(x[None], w[None], stride)
        pt = dict(size=size, k=k, stride=stride, c=ch, s=s, ms=ms, ws=ws,
                  mixed=bool(len(sweep) % 2),
                  ptr=r.checksum(e["ptr"].view(np.float32)),
                  offsets=r.checksum(e["offsets"].view(np.float32)),
                  f_data=r.checksum(e["f_data"]), k_data=r.checksum(e["k_data"]),
                  ecr=r.checksum(y), ecr_ops=list(eops))
        for ps in (1, 2):
            try:
                r.pack_count(size, k, stride, 2, ps)
            except OracleError:
                continue
            pf = r.pecr_convert(x, w, stride, 2, 2, ps)
            pmax, pops = r.pecr_conv(x[None], w[None], stride, 2, 2, ps, 0)
            pmean, _ = r.pecr_conv(x[None], w[None], stride, 2, 2, ps, 1)
            pt[f"pecr_ps{ps}"] = dict(
                count=r.checksum(pf["count"].view(np.float32)),
                start=r.checksum(pf["pack_start"].view(np.float32)),
                data=r.checksum(pf["data"]), index=r.checksum(pf["index"].view(np.float32)),
                max=r.checksum(pmax), mean=r.checksum(pmean), ops=list(pops))
        sweep.append(pt)
    g["sweep"] = sweep

    with open(OUT, "w") as f:
        json.dump(g, f, indent=1)
    print("wrote", OUT, len(sweep), "sweep points")


if __name__ == "__main__":
    main()
