"""Generate tests/golden/forward_vectors.json by running the UNMODIFIED
reference forward() (src/pipeline.cpp:212-301, through oracle/ref_bridge.cpp)
on the seeded networks of tests/forward_nets.py.  Dev container only:

    make -C oracle ref && python tests/golden/make_golden_forward.py
"""
import json
import os
import sys

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), "..", ".."))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from forward_nets import BAD_PECR, NETS, build  # noqa: E402
from oracle.oracle import OracleError, RefLib  # noqa: E402

OUT = os.path.join(os.path.dirname(__file__), "forward_vectors.json")


def main() -> None:
    r = RefLib()
    g = {"source": "sconv_ref::forward of oracle/_ref/libsconv_ref.so", "nets": {}}
    for name, spec in NETS.items():
        for img in range(2):
            x, layers = build(r, spec, img)
            for method in (0, 1, 2):
                y, lo, co, ops, fb = r.forward(x, layers, method)
                g["nets"][f"{name}/{img}/{method}"] = {
                    "layer_outputs": [r.checksum(v) for v in lo],
                    "conv_outputs": [None if v is None else r.checksum(v) for v in co],
                    "shape": list(y.shape), "ops": list(ops), "fallback": fb}
    x, layers = build(r, BAD_PECR, 0)
    try:
        r.forward(x, layers, 2)
        raise SystemExit("BAD_PECR did not fail")
    except OracleError as e:
        g["bad_pecr"] = {"code": e.code, "msg": str(e)}
    with open(OUT, "w") as f:
        json.dump(g, f, indent=1)
    print("wrote", OUT, len(g["nets"]), "cases")


if __name__ == "__main__":
    main()
