"""Pin the C oracle (oracle/sconv_oracle.c) before trusting it.

1. against the golden vectors produced by the UNMODIFIED reference
   (tests/golden/reference_vectors.json, tests/golden/make_golden.py), and
2. directly against the reference library (oracle/_ref) on fresh seeded
   inputs, when that library is present.
"""
import numpy as np
import pytest

from oracle.oracle import OracleError


def test_rng_vectors(orc, golden):
    for seed, vals in golden["rng"].items():
        assert ["%016x" % v for v in orc.rng(int(seed), 5)] == vals
    # frozen vectors of test_dataset.cpp:43-48
    assert orc.rng(42, 3) == [0x15780b2e0c2ec716, 0x6104d9866d113a7e, 0xae17533239e499a1]


def test_generate(orc, golden):
    for g in golden["generate"]:
        m = orc.generate(g["h"], g["w"], g["c"], g["s"], g["seed"])
        assert orc.checksum(m) == g["checksum"]
        assert int((m == 0).sum()) == g["zeros"]
    assert int((orc.generate(32, 32, 1, 0.7, 42) == 0).sum()) == 716


def test_fixtures(orc, golden):
    fx = golden["fixtures"]
    f5 = np.array(fx["f5"], np.float32).reshape(1, 5, 5)
    k3 = np.array(fx["k3"], np.float32).reshape(1, 3, 3)
    dense, ops = orc.dense_conv(f5, k3, 1)
    assert dense.reshape(-1).tolist() == fx["dense"] == [51, 49, 61, 83, 70, 75, 93, 106, 103]
    assert list(ops) == fx["dense_ops"]
    e = orc.ecr_convert(f5, k3, 1)
    assert e["ptr"].reshape(-1).tolist() == fx["ecr_ptr"]
    assert e["offsets"].reshape(-1).tolist() == fx["ecr_offsets"]
    assert e["f_data"].reshape(-1).tolist() == fx["ecr_f"]
    assert e["k_data"].reshape(-1).tolist() == fx["ecr_k"]
    y, ops = orc.ecr_spmv(e["ptr"], e["f_data"], e["k_data"])
    assert y.reshape(-1).tolist() == fx["dense"]
    assert ops == (27, 18)  # test_ecr.cpp:107-116
    p = orc.pecr_convert(f5, 3, 3, 1, 2, 2, 1)
    assert p["count"].reshape(-1).tolist() == fx["pecr_count"]
    assert p["pack_start"].tolist() == fx["pecr_start"]
    assert p["data"].tolist() == fx["pecr_data"]
    assert p["index"].tolist() == fx["pecr_index"]
    pooled, pops = orc.pecr_conv_pool(p, k3, 2, 2, 0)
    assert pooled.reshape(-1).tolist() == fx["pecr_max"] == [83, 75, 106, 106]
    assert list(pops) == fx["pecr_ops"]
    mean, _ = orc.pecr_conv_pool(p, k3, 2, 2, 1)
    assert mean.reshape(-1).tolist() == fx["pecr_mean"]
    pb, _ = orc.pecr_conv(f5[None], k3[None], 1, 2, 2, 1, 0)
    assert pb.reshape(-1).tolist() == fx["pecr_max"]


def test_kats(orc, golden):
    for k in golden["kats"]:
        x = orc.generate(k["h"], k["h"], k["c"], k["s"], k["ms"])
        w = orc.generate(3, 3, k["c"], 0.0, k["ws"]) - np.float32(0.5)
        assert orc.checksum(x) == k["map"]
        y, ops = orc.ecr_conv(x[None], w[None], 1)
        assert orc.checksum(y) == k["ecr"] and list(ops) == k["ecr_ops"]
        p, pops = orc.pecr_conv(x[None], w[None], 1, 2, 2, 2, 0)
        assert orc.checksum(p) == k["pecr"] and list(pops) == k["pecr_ops"]


def test_pack_count(orc, golden):
    for case in golden["pack_count"]:
        if "packs" in case:
            assert orc.pack_count(*case["args"]) == case["packs"]
        else:
            with pytest.raises(OracleError) as ei:
                orc.pack_count(*case["args"])
            assert ei.value.kind == case["error"]


def _sweep_inputs(orc, pt):
    x = orc.generate(pt["size"], pt["size"], pt["c"], pt["s"], pt["ms"])
    w = orc.generate(pt["k"], pt["k"], pt["c"], 0.0, pt["ws"])
    if pt["mixed"]:
        w = w - np.float32(0.5)
    return x, w


def test_sweep(orc, golden):
    for pt in golden["sweep"]:
        x, w = _sweep_inputs(orc, pt)
        e = orc.ecr_convert(x, w, pt["stride"])
        assert orc.checksum(e["ptr"].view(np.float32)) == pt["ptr"]
        assert orc.checksum(e["offsets"].view(np.float32)) == pt["offsets"]
        assert orc.checksum(e["f_data"]) == pt["f_data"]
        assert orc.checksum(e["k_data"]) == pt["k_data"]
        y, ops = orc.ecr_conv(x[None], w[None], pt["stride"])
        assert orc.checksum(y) == pt["ecr"] and list(ops) == pt["ecr_ops"]
        y2, ops2 = orc.ecr_spmv(e["ptr"], e["f_data"], e["k_data"])
        assert orc.checksum(y2) == pt["ecr"] and list(ops2) == pt["ecr_ops"]
        for ps in (1, 2):
            key = f"pecr_ps{ps}"
            if key not in pt:
                continue
            g = pt[key]
            p = orc.pecr_convert(x, pt["k"], pt["k"], pt["stride"], 2, 2, ps)
            assert orc.checksum(p["count"].view(np.float32)) == g["count"]
            assert orc.checksum(p["pack_start"].view(np.float32)) == g["start"]
            assert orc.checksum(p["data"]) == g["data"]
            assert orc.checksum(p["index"].view(np.float32)) == g["index"]
            pm, pops = orc.pecr_conv_pool(p, w, 2, 2, 0)
            assert orc.checksum(pm) == g["max"] and list(pops) == g["ops"]
            pmean, _ = orc.pecr_conv_pool(p, w, 2, 2, 1)
            assert orc.checksum(pmean) == g["mean"]
            pb, _ = orc.pecr_conv(x[None], w[None], pt["stride"], 2, 2, ps, 0)
            assert orc.checksum(pb) == g["max"]


def test_format_errors(orc):
    x = orc.generate(5, 5, 1, 0.5, 1)
    w = orc.generate(3, 3, 1, 0.0, 2)
    e = orc.ecr_convert(x, w, 1)
    ptr = e["ptr"].copy()
    ptr[1, 1] = -2
    with pytest.raises(OracleError) as ei:
        orc.ecr_spmv(ptr, e["f_data"], e["k_data"])
    assert ei.value.kind == "FormatError"
    ptr[1, 1] = 10
    with pytest.raises(OracleError):
        orc.ecr_spmv(ptr, e["f_data"], e["k_data"])


@pytest.mark.parametrize("seed", range(6))
def test_against_reference_library(orc, ref, seed):
    """Fresh random shapes: C oracle == the reference itself, bit for bit."""
    rng = np.random.default_rng(seed)
    size = int(rng.integers(5, 30))
    k = int(rng.choice([1, 2, 3, 5]))
    k = min(k, size)
    stride = int(rng.integers(1, 4))
    c = int(rng.integers(1, 6))
    s = float(rng.choice([0.0, 0.3, 0.7, 0.95, 1.0]))
    x = ref.generate(size, size + 1, c, s, seed * 7 + 1)
    w = ref.generate(k, k, c, 0.0, seed * 7 + 2) - np.float32(0.5)
    assert orc.checksum(orc.generate(size, size + 1, c, s, seed * 7 + 1)) == ref.checksum(x)
    y_r, ops_r = ref.ecr_conv(x[None], w[None], stride)
    y_o, ops_o = orc.ecr_conv(x[None], w[None], stride)
    assert ref.checksum(y_r) == orc.checksum(y_o) and ops_r == ops_o
    d_r, dops_r = ref.dense_conv(x, w, stride)
    d_o, dops_o = orc.dense_conv(x, w, stride)
    assert ref.checksum(d_r) == orc.checksum(d_o) and dops_r == dops_o
    e_r = ref.ecr_convert(x, w, stride, workers=3)
    e_o = orc.ecr_convert(x, w, stride)
    for key in ("ptr", "offsets", "f_data", "k_data"):
        assert np.array_equal(e_r[key].view(np.uint32), e_o[key].view(np.uint32)), key
    assert np.array_equal(ref.window_nnz(x, k, k, stride), orc.window_nnz(x, k, k, stride))
    for ps in (1, 2):
        for pw in (1, 2, 3):
            try:
                ref.pack_count(size + 1, k, stride, pw, ps)
                ref.pack_count(size, k, stride, pw, ps)
            except OracleError:
                continue
            for mode in (0, 1):
                p_r, pops_r = ref.pecr_conv(x[None], w[None], stride, pw, pw, ps, mode)
                p_o, pops_o = orc.pecr_conv(x[None], w[None], stride, pw, pw, ps, mode)
                assert ref.checksum(p_r) == orc.checksum(p_o) and pops_r == pops_o
            f_r = ref.pecr_convert(x, w, stride, pw, pw, ps)
            f_o = orc.pecr_convert(x, k, k, stride, pw, pw, ps)
            for key in ("count", "pack_start", "data", "index"):
                assert np.array_equal(np.asarray(f_r[key]), np.asarray(f_o[key])), key
