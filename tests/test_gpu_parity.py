"""Parity of the CUDA path (through the C ABI) with the reference.

Checker: the C oracle (pinned to the reference by tests/test_oracle.py) and
the golden vectors of the unmodified reference.  Bars:

* index / count / format arrays: bit-exact;
* EXACT arithmetic (default): outputs bit-exact;
* FAST arithmetic (FFMA): |gpu - ref| <= ATOL + RTOL*|ref| with ATOL = RTOL
  = 1e-5 (north_star: "within rel 1e-5 / abs 1e-5").
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ATOL = 1e-5
RTOL = 1e-5


def bits_equal(a, b):
    a = np.ascontiguousarray(a, np.float32)
    b = np.ascontiguousarray(b, np.float32)
    return a.shape == b.shape and np.array_equal(a.view(np.uint32), b.view(np.uint32))


def close(a, b):
    return np.all(np.abs(a.astype(np.float64) - b) <= ATOL + RTOL * np.abs(b.astype(np.float64)))


def inputs(orc, n, c, h, w, k, kh, kw, s, seed, mixed=True):
    x = np.stack([orc.generate(h, w, c, s, seed + i) for i in range(n)])
    f = np.stack([orc.generate(kh, kw, c, 0.0, seed + 1000 + j) for j in range(k)])
    if mixed:
        f = f - np.float32(0.5)
    return x, f


# ---------------------------------------------------------------------------
# two-phase API: formats bit-exact
# ---------------------------------------------------------------------------

def test_fixture_f5(sc, golden):
    fx = golden["fixtures"]
    f5 = sc.FeatureMap(1, 5, 5, fx["f5"])
    k3 = sc.Filter(1, 3, 3, fx["k3"])
    e = sc.ecr_convert(f5, k3, sc.ConvConfig(1))
    assert np.concatenate([r.ptr for r in e.block_rows]).tolist() == fx["ecr_ptr"]
    assert np.concatenate([r.offsets for r in e.block_rows]).tolist() == fx["ecr_offsets"]
    assert np.concatenate([r.f_data for r in e.block_rows]).tolist() == fx["ecr_f"]
    assert np.concatenate([r.k_data for r in e.block_rows]).tolist() == fx["ecr_k"]
    ops = sc.OpCount()
    out = sc.ecr_spmv_conv(e, ops)
    assert out.values.tolist() == fx["dense"] and (ops.multiplications, ops.additions) == (27, 18)
    pool = sc.PoolConfig(2, 2, 1, sc.PoolMode.kMax)
    p = sc.pecr_convert(f5, k3, sc.ConvConfig(1), pool)
    assert np.concatenate([pk.count for row in p.pool_rows for pk in row]).tolist() == fx["pecr_count"]
    assert np.concatenate([pk.data for row in p.pool_rows for pk in row]).tolist() == fx["pecr_data"]
    assert np.concatenate([pk.index for row in p.pool_rows for pk in row]).tolist() == fx["pecr_index"]
    pops = sc.OpCount()
    pooled = sc.pecr_conv_pool(p, pops)
    assert pooled.values.tolist() == [83, 75, 106, 106]
    assert [pops.multiplications, pops.additions] == fx["pecr_ops"]
    p.dims.pool.mode = sc.PoolMode.kMean
    assert sc.pecr_conv_pool(p).values.tolist() == fx["pecr_mean"]
    # the fused entries agree with the frozen values too
    y = sc.pecr_conv_pool_batched(f5.array()[None], k3.array()[None], 1, pool)
    assert y.reshape(-1).tolist() == [83, 75, 106, 106]
    y = sc.ecr_conv_batched(f5.array()[None], k3.array()[None], 1)
    assert y.reshape(-1).tolist() == fx["dense"]


def test_golden_sweep_formats_and_outputs(sc, orc, golden):
    for pt in golden["sweep"]:
        x = orc.generate(pt["size"], pt["size"], pt["c"], pt["s"], pt["ms"])
        w = orc.generate(pt["k"], pt["k"], pt["c"], 0.0, pt["ws"])
        if pt["mixed"]:
            w = w - np.float32(0.5)
        m = sc.FeatureMap(pt["c"], pt["size"], pt["size"], x)
        f = sc.Filter(pt["c"], pt["k"], pt["k"], w)
        cfg = sc.ConvConfig(pt["stride"])
        e = sc.ecr_convert(m, f, cfg)
        cat = lambda key: np.concatenate([getattr(r, key) for r in e.block_rows])
        assert orc.checksum(cat("ptr").view(np.float32)) == pt["ptr"]
        assert orc.checksum(cat("offsets").view(np.float32)) == pt["offsets"]
        assert orc.checksum(cat("f_data")) == pt["f_data"]
        assert orc.checksum(cat("k_data")) == pt["k_data"]
        ops = sc.OpCount()
        y = sc.ecr_spmv_conv(e, ops)
        assert orc.checksum(y.values) == pt["ecr"]
        assert [ops.multiplications, ops.additions] == pt["ecr_ops"]
        ops = sc.OpCount()
        yb = sc.ecr_conv_batched(x[None], w[None], pt["stride"], counters=ops)
        assert orc.checksum(yb) == pt["ecr"]
        assert [ops.multiplications, ops.additions] == pt["ecr_ops"]
        for ps in (1, 2):
            g = pt.get(f"pecr_ps{ps}")
            if g is None:
                continue
            pool = sc.PoolConfig(2, 2, ps, sc.PoolMode.kMax)
            p = sc.pecr_convert(m, f, cfg, pool)
            packs = [pk for row in p.pool_rows for pk in row]
            assert orc.checksum(np.concatenate([pk.count for pk in packs]).view(np.float32)) == g["count"]
            assert orc.checksum(np.concatenate([pk.data for pk in packs] + [np.zeros(0, np.float32)])) == g["data"]
            assert orc.checksum(np.concatenate([pk.index for pk in packs] + [np.zeros(0, np.int32)]).view(np.float32)) == g["index"]
            pops = sc.OpCount()
            assert orc.checksum(sc.pecr_conv_pool(p, pops).values) == g["max"]
            assert [pops.multiplications, pops.additions] == g["ops"]
            pops = sc.OpCount()
            yb = sc.pecr_conv_pool_batched(x[None], w[None], pt["stride"], pool, counters=pops)
            assert orc.checksum(yb) == g["max"]
            assert [pops.multiplications, pops.additions] == g["ops"]
            mean = sc.PoolConfig(2, 2, ps, sc.PoolMode.kMean)
            assert orc.checksum(sc.pecr_conv_pool_batched(x[None], w[None], pt["stride"], mean)) == g["mean"]


def test_kats(sc, orc, golden):
    for k in golden["kats"]:
        x = orc.generate(k["h"], k["h"], k["c"], k["s"], k["ms"])
        w = orc.generate(3, 3, k["c"], 0.0, k["ws"]) - np.float32(0.5)
        assert sc.checksum_hex(sc.generate(k["h"], k["h"], k["c"], k["s"], k["ms"]).values) == k["map"]
        ops = sc.OpCount()
        y = sc.ecr_conv_batched(x[None], w[None], 1, counters=ops)
        assert sc.checksum_hex(y) == k["ecr"]
        assert [ops.multiplications, ops.additions] == k["ecr_ops"]
        ops = sc.OpCount()
        p = sc.pecr_conv_pool_batched(x[None], w[None], 1, sc.PoolConfig(2, 2, 2), counters=ops)
        assert sc.checksum_hex(p) == k["pecr"]
        assert [ops.multiplications, ops.additions] == k["pecr_ops"]


# ---------------------------------------------------------------------------
# fused batched path: tiled + generic kernels, EXACT bitwise, FAST tolerance
# ---------------------------------------------------------------------------

SHAPES = [
    # n, c, h, w, k, kh, kw, stride, sparsity        (tiled: 3x3 s1, K >= 32)
    (2, 3, 18, 20, 64, 3, 3, 1, 0.7),
    (2, 13, 19, 23, 128, 3, 3, 1, 0.7),
    (1, 64, 30, 30, 256, 3, 3, 1, 0.9),
    (3, 17, 16, 34, 96, 3, 3, 1, 0.5),
    (1, 8, 10, 10, 40, 3, 3, 1, 0.0),
    (2, 9, 12, 12, 128, 3, 3, 1, 1.0),
    (1, 5, 40, 9, 64, 3, 3, 1, 0.8),
    # generic shapes
    (2, 4, 11, 11, 7, 5, 5, 1, 0.7),
    (2, 3, 17, 15, 5, 3, 3, 2, 0.5),
    (1, 2, 12, 13, 3, 2, 2, 3, 0.6),
    (1, 20, 11, 11, 50, 5, 5, 1, 0.7),   # LeNet conv2 shape
    (2, 6, 9, 9, 33, 1, 1, 1, 0.7),
    (1, 3, 8, 8, 16, 3, 3, 1, 0.7),     # K < 32 -> generic
]


@pytest.mark.parametrize("shape", SHAPES, ids=[str(s) for s in SHAPES])
def test_ecr_fused(sc, orc, shape):
    n, c, h, w, k, kh, kw, s, sp = shape
    x, f = inputs(orc, n, c, h, w, k, kh, kw, sp, seed=hash(shape) & 0xFFFF)
    ref, rops = orc.ecr_conv(x, f, s)
    for generic in (False, True):
        ops = sc.OpCount()
        y = sc.ecr_conv_batched(x, f, s, counters=ops, generic=generic)
        assert bits_equal(y, ref), f"EXACT mismatch generic={generic}"
        assert (ops.multiplications, ops.additions) == rops
        yf = sc.ecr_conv_batched(x, f, s, fast=True, generic=generic)
        assert close(yf, ref)
    # empty windows produce +0.0 (ptr == -1 law)
    nnz = np.stack([orc.window_nnz(x[i], kh, kw, s) for i in range(n)])
    empty = np.broadcast_to(nnz[:, None] == 0, ref.shape)
    assert not np.signbit(y[empty]).any() and not y[empty].any()


PSHAPES = [
    # n, c, h, w, k, kh, kw, stride, pw, ph, ps, sparsity
    (2, 3, 18, 22, 64, 3, 3, 1, 2, 2, 2, 0.7),    # tiled P=2
    (2, 19, 34, 34, 128, 3, 3, 1, 2, 2, 2, 0.7),
    (1, 64, 16, 16, 256, 3, 3, 1, 2, 2, 2, 0.9),
    (2, 5, 30, 14, 72, 3, 3, 1, 2, 2, 2, 0.5),
    (2, 3, 9, 9, 5, 3, 3, 1, 2, 2, 1, 0.6),       # overlapping pool -> generic
    (1, 4, 13, 13, 6, 3, 3, 2, 2, 2, 2, 0.7),
    (1, 2, 13, 13, 4, 3, 3, 1, 3, 3, 2, 0.5),
    (1, 3, 9, 9, 40, 3, 3, 1, 1, 1, 1, 0.7),
]


@pytest.mark.parametrize("shape", PSHAPES, ids=[str(s) for s in PSHAPES])
def test_pecr_fused(sc, orc, shape):
    n, c, h, w, k, kh, kw, s, pw, ph, ps, sp = shape
    x, f = inputs(orc, n, c, h, w, k, kh, kw, sp, seed=hash(shape) & 0xFFFF)
    for mode in (0, 1):
        ref, rops = orc.pecr_conv(x, f, s, pw, ph, ps, mode)
        pool = sc.PoolConfig(pw, ph, ps, sc.PoolMode(mode))
        for generic in (False, True):
            ops = sc.OpCount()
            y = sc.pecr_conv_pool_batched(x, f, s, pool, counters=ops, generic=generic)
            assert bits_equal(y, ref), f"EXACT mismatch mode={mode} generic={generic}"
            assert (ops.multiplications, ops.additions) == rops
            yf = sc.pecr_conv_pool_batched(x, f, s, pool, fast=True, generic=generic)
            assert close(yf, ref)
        # PECR == pool(relu(conv)) (test_pecr.cpp:35-42)
        if mode == 0:
            conv, _ = orc.ecr_conv(x, f, s)
            sep = np.stack([orc.pool(orc.relu(conv[i]), pw, ph, ps, 0) for i in range(n)])
            assert bits_equal(y, sep)


# ---------------------------------------------------------------------------
# every tiled configuration, forced (SCONV_F_KERNEL), including the v3
# warp-specialised kernel on K = 512 / 14-wide maps and ragged tile lists
# ---------------------------------------------------------------------------

KSHAPES = [
    # n, c, h, w, k, sparsity
    (2, 13, 16, 16, 512, 0.7),     # conv5-like 14x14, K tail-free
    (3, 9, 30, 30, 160, 0.7),      # 28x28, K not a multiple of 128 (tail CTA)
    (1, 11, 11, 19, 96, 0.5),      # ragged tiles in both directions
    (2, 6, 10, 13, 64, 0.9),
    (1, 5, 12, 12, 256, 1.0),      # all zero
    (1, 7, 9, 9, 128, 0.0),        # dense
]
KERNELS = [1, 2, 3, 4, 5, 6, "A", "B", "C", "D", "E", "F", "G", "P", "U", "V", "W"]


@pytest.mark.parametrize("kid", KERNELS, ids=[str(k) for k in KERNELS])
@pytest.mark.parametrize("shape", KSHAPES, ids=[str(s) for s in KSHAPES])
def test_forced_kernels(sc, orc, shape, kid):
    n, c, h, w, k, sp = shape
    x, f = inputs(orc, n, c, h, w, k, 3, 3, sp, seed=(hash(shape) ^ 77) & 0xFFFF)
    ref, _ = orc.ecr_conv(x, f, 1)
    y = sc.ecr_conv_batched(x, f, 1, kernel=kid)
    assert bits_equal(y, ref), f"ECR EXACT mismatch kernel={kid}"
    assert close(sc.ecr_conv_batched(x, f, 1, fast=True, kernel=kid), ref)
    if kid in ("B", "U", "V") or (h - 2) % 2 or (w - 2) % 2:  # ECR-only configs
        return
    for mode in (0, 1):
        pref, _ = orc.pecr_conv(x, f, 1, 2, 2, 2, mode)
        pool = sc.PoolConfig(2, 2, 2, sc.PoolMode(mode))
        p = sc.pecr_conv_pool_batched(x, f, 1, pool, kernel=kid)
        assert bits_equal(p, pref), f"PECR EXACT mismatch kernel={kid} mode={mode}"
        assert close(sc.pecr_conv_pool_batched(x, f, 1, pool, fast=True, kernel=kid), pref)


@pytest.mark.parametrize("n", [8, 9, 35])
def test_host_pointer_pipeline(sc, orc, n):
    """Host-pointer calls with n >= 8 run as image chunks alternating between
    two streams (H2D / compute / D2H overlap); results, counters and the
    ragged last chunk must match the oracle exactly."""
    c, h, w, k = 5, 12, 14, 64
    x, f = inputs(orc, n, c, h, w, k, 3, 3, 0.7, seed=4242 + n)
    ops = sc.OpCount()
    y = sc.ecr_conv_batched(x, f, 1, counters=ops)
    ref, rops = orc.ecr_conv(x, f, 1)
    assert bits_equal(y, ref)
    assert (ops.multiplications, ops.additions) == rops
    ops = sc.OpCount()
    p = sc.pecr_conv_pool_batched(x, f, 1, sc.PoolConfig(2, 2, 2), counters=ops)
    pref, pops = orc.pecr_conv(x, f, 1, 2, 2, 2, 0)
    assert bits_equal(p, pref)
    assert (ops.multiplications, ops.additions) == pops


def test_errors(sc):
    x = np.ones((1, 2, 5, 5), np.float32)
    with pytest.raises(sc.ShapeError):
        sc.ecr_conv_batched(x, np.ones((3, 1, 3, 3), np.float32))
    with pytest.raises(sc.ShapeError):
        sc.ecr_conv_batched(np.ones((1, 1, 3, 3), np.float32), np.ones((1, 1, 5, 5), np.float32))
    with pytest.raises(sc.ConfigError):
        sc.ecr_conv_batched(x, np.ones((1, 2, 3, 3), np.float32), 0)
    with pytest.raises(sc.ConfigError):  # 7x7, k3 -> 5 wide, pool 2 stride 2 dangles
        sc.pecr_conv_pool_batched(np.ones((1, 1, 7, 7), np.float32),
                                  np.ones((1, 1, 3, 3), np.float32), 1, sc.PoolConfig(2, 2, 2))
    with pytest.raises(sc.ShapeError):
        sc.ecr_convert(sc.FeatureMap(2, 5, 5), sc.Filter(1, 3, 3, np.ones(9)))


def test_corrupted_formats(sc, orc):
    """test_ecr.cpp:119-137, test_pecr.cpp:161-166."""
    m = sc.FeatureMap(1, 5, 5, orc.generate(5, 5, 1, 0.5, 3))
    f = sc.Filter(1, 3, 3, np.arange(1, 10))
    e = sc.ecr_convert(m, f)
    e.block_rows[1].ptr[1] = -2
    with pytest.raises(sc.FormatError):
        sc.ecr_spmv_conv(e)
    e.block_rows[1].ptr[1] = 10
    with pytest.raises(sc.FormatError):
        sc.ecr_spmv_conv(e)
    e = sc.ecr_convert(m, f)
    e.block_rows.pop()
    with pytest.raises(sc.FormatError):
        sc.ecr_spmv_conv(e)
    e = sc.ecr_convert(m, f)
    e.block_rows[0].f_data = e.block_rows[0].f_data[:-1]
    with pytest.raises(sc.FormatError):
        sc.ecr_spmv_conv(e)
    p = sc.pecr_convert(m, f, sc.ConvConfig(1), sc.PoolConfig(2, 2, 1))
    p.pool_rows[0][0].data = np.append(p.pool_rows[0][0].data, np.float32(1))
    with pytest.raises(sc.FormatError):
        sc.pecr_conv_pool(p)
    p = sc.pecr_convert(m, f, sc.ConvConfig(1), sc.PoolConfig(2, 2, 1))
    if len(p.pool_rows[0][0].index):
        p.pool_rows[0][0].index[0] = 99
        with pytest.raises(sc.FormatError):
            sc.pecr_conv_pool(p)


def test_sentinel_law(sc):
    """test_ecr.cpp:139-155: one nonzero -> one window with ptr 1, rest -1 / +0.0."""
    m = sc.FeatureMap(1, 6, 6)
    m.values[0] = 2.5
    f = sc.Filter(1, 3, 3, np.arange(1, 10))
    e = sc.ecr_convert(m, f)
    ptr = np.stack([r.ptr for r in e.block_rows])
    expect = -np.ones((4, 4), np.int32)
    expect[0, 0] = 1
    assert np.array_equal(ptr, expect)
    out = sc.ecr_spmv_conv(e).array()[0]
    assert out[0, 0] == 2.5 and not np.signbit(out).any() and (out[1:] == 0).all()


def test_all_zero_map(sc):
    """acceptance criterion 9 (acceptance_main.cpp:426-475)."""
    x = np.zeros((2, 3, 16, 16), np.float32)
    w = np.random.default_rng(0).random((64, 3, 3, 3), np.float32) - 0.5
    for fn, args in ((sc.ecr_conv_batched, ()), (sc.pecr_conv_pool_batched, (sc.PoolConfig(2, 2, 2),))):
        ops = sc.OpCount()
        y = fn(x, w, 1, *args, counters=ops)
        assert not y.any() and not np.signbit(y).any()
        assert ops.multiplications == 0 and ops.additions == 0
    e = sc.ecr_convert(sc.FeatureMap(3, 16, 16), sc.Filter(3, 3, 3, w[0]))
    assert all((r.ptr == -1).all() for r in e.block_rows)


def test_windows_reconstruct(sc, orc):
    """Lossless windows (test_ecr.cpp:198-206, test_pecr.cpp:219-229)."""
    x = orc.generate(13, 13, 3, 0.7, 11)
    m = sc.FeatureMap(3, 13, 13, x)
    f = sc.Filter(3, 3, 3, orc.generate(3, 3, 3, 0.0, 12))
    e = sc.ecr_convert(m, f, sc.ConvConfig(2))
    for b in range(e.dims.out_h()):
        for t in range(e.dims.out_w()):
            assert np.array_equal(sc.ecr_window(e, b, t), x[:, 2 * b:2 * b + 3, 2 * t:2 * t + 3].reshape(-1))
    p = sc.pecr_convert(m, f, sc.ConvConfig(1), sc.PoolConfig(2, 2, 1))
    for b in range(p.packs_h()):
        for t in range(p.packs_w()):
            for n in range(4):
                wy, wx = b + n // 2, t + n % 2
                assert np.array_equal(sc.pecr_window(p, b, t, n), x[:, wy:wy + 3, wx:wx + 3].reshape(-1))


def test_multichannel_conv(sc, orc):
    x = orc.generate(12, 12, 4, 0.6, 5)
    fs = [sc.Filter(4, 3, 3, orc.generate(3, 3, 4, 0.0, 100 + i) - np.float32(0.5)) for i in range(40)]
    out = sc.multichannel_conv(sc.FeatureMap(4, 12, 12, x), fs, sc.ConvConfig(1))
    ref, _ = orc.ecr_conv(x[None], np.stack([f.array() for f in fs]), 1)
    assert bits_equal(out.array(), ref[0])


def test_torch_device_path(sc, orc):
    torch = pytest.importorskip("torch")
    x, f = inputs(orc, 2, 16, 20, 20, 128, 3, 3, 0.7, seed=77)
    ref, _ = orc.ecr_conv(x, f, 1)
    xd, fd = torch.from_numpy(x).cuda(), torch.from_numpy(f).cuda()
    y = sc.ecr_conv_batched(xd, fd, 1)
    torch.cuda.synchronize()
    assert bits_equal(y.cpu().numpy(), ref)
    y2 = sc.ecr_conv_batched(xd, fd, 1, sync=False)
    torch.cuda.synchronize()
    assert bits_equal(y2.cpu().numpy(), ref)
    p = sc.pecr_conv_pool_batched(xd, fd, 1, sc.PoolConfig(2, 2, 2))
    pref, _ = orc.pecr_conv(x, f, 1, 2, 2, 2, 0)
    assert bits_equal(p.cpu().numpy(), pref)


def test_determinism(sc, orc):
    x, f = inputs(orc, 2, 32, 30, 30, 128, 3, 3, 0.7, seed=3)
    a = sc.ecr_conv_batched(x, f, 1, fast=True)
    for _ in range(3):
        assert bits_equal(sc.ecr_conv_batched(x, f, 1, fast=True), a)


# ---------------------------------------------------------------------------
# full-size VGG-19 layers: sampled (image, filter) pairs against the oracle
# ---------------------------------------------------------------------------
VGG_FULL = [("conv1_1", 3, 64, 224, False), ("conv1_2", 64, 64, 224, True),
            ("conv2_2", 128, 128, 112, True), ("conv3_2", 256, 256, 56, False),
            ("conv4_4", 512, 512, 28, True), ("conv5_1", 512, 512, 14, False)]


@pytest.mark.parametrize("layer", VGG_FULL, ids=[v[0] for v in VGG_FULL])
def test_vgg_full_size_sampled(sc, orc, layer):
    """Full layer on the GPU (N=2, all K filters, reference generator inputs,
    sparsity 0.7); filters {0, 1, K/2, K-1} of both images checked against the
    oracle: EXACT bit-exact, FAST within 1e-5 + 1e-5|ref|."""
    name, C, K, H, pooled = layer
    l = [v[0] for v in VGG_FULL].index(name)
    x = sc.generate_batch([1000 * l + n for n in range(2)], H + 2, H + 2, C, 0.7)
    w = sc.generate_batch([5000 * l + k for k in range(K)], 3, 3, C, 0.0) - np.float32(0.5)
    ks = [0, 1, K // 2, K - 1]
    pool = sc.PoolConfig(2, 2, 2)
    for fast in (False, True):
        if pooled:
            y = sc.pecr_conv_pool_batched(x, w, 1, pool, fast=fast)
            ref, _ = orc.pecr_conv(x, w[ks], 1, 2, 2, 2, 0)
        else:
            y = sc.ecr_conv_batched(x, w, 1, fast=fast)
            ref, _ = orc.ecr_conv(x, w[ks], 1)
        got = y[:, ks]
        if fast:
            assert close(got, ref)
        else:
            assert bits_equal(got, ref)


# ---------------------------------------------------------------------------
# the v3 kernel instantiated for 1x1 and 5x5 windows (GoogLeNet / LeNet
# layers of BASELINE config 2), default selection and forced
# ---------------------------------------------------------------------------

WSHAPES = [
    # n, c, h, w, k, kh, sparsity
    (2, 20, 11, 11, 50, 5, 0.95),   # LeNet conv2
    (2, 32, 14, 14, 128, 5, 0.9),   # GoogLeNet 4e 5x5 branch
    (2, 48, 12, 13, 96, 5, 0.5),    # ragged tiles
    (2, 37, 14, 14, 192, 1, 0.9),   # GoogLeNet 4a 1x1 branch
    (1, 19, 7, 9, 64, 1, 0.7),      # 1x1, K < 128, ragged
    (1, 8, 10, 10, 256, 1, 0.0),    # 1x1 dense
]


@pytest.mark.parametrize("shape", WSHAPES, ids=[str(s) for s in WSHAPES])
def test_ws_1x1_5x5(sc, orc, shape):
    n, c, h, w, k, kk, sp = shape
    x, f = inputs(orc, n, c, h, w, k, kk, kk, sp, seed=(hash(shape) ^ 91) & 0xFFFF)
    ref, rops = orc.ecr_conv(x, f, 1)
    plan = sc.launch_plan(n, c, h, w, k, kk, kk, 1)
    # 5x5: 4x4 tiles, or 2x2 tiles when those fit in one wave (small grids);
    # 1x1: the dense ordered GEMM (pointwise.cuh)
    assert plan["kernel"] in ((110, 117) if kk == 5 else (401, 402, 108, 109, 114, 115))
    ops = sc.OpCount()
    y = sc.ecr_conv_batched(x, f, 1, counters=ops)
    assert bits_equal(y, ref)
    assert (ops.multiplications, ops.additions) == rops
    assert close(sc.ecr_conv_batched(x, f, 1, fast=True), ref)
    both = ("J", "Q") if kk == 5 else (("H", "N") if k >= 128 else ("I", "O"))
    for forced in both:
        assert bits_equal(sc.ecr_conv_batched(x, f, 1, kernel=forced), ref), forced
        assert close(sc.ecr_conv_batched(x, f, 1, fast=True, kernel=forced), ref), forced
    if (h - kk + 1) % 2 == 0 and (w - kk + 1) % 2 == 0:
        for mode in (0, 1):
            pref, _ = orc.pecr_conv(x, f, 1, 2, 2, 2, mode)
            pool = sc.PoolConfig(2, 2, 2, sc.PoolMode(mode))
            assert bits_equal(sc.pecr_conv_pool_batched(x, f, 1, pool), pref)
            assert close(sc.pecr_conv_pool_batched(x, f, 1, pool, fast=True), pref)
            for forced in both:
                assert bits_equal(sc.pecr_conv_pool_batched(x, f, 1, pool, kernel=forced), pref)
    with pytest.raises(ValueError):  # SCONV_ERR_ARG: a 3x3 config forced on a 1x1/5x5 shape
        sc.ecr_conv_batched(x, f, 1, kernel="A")
    if kk == 1:
        assert bits_equal(sc.ecr_conv_batched(x, f, 1, kernel="Y"), ref)
    else:
        with pytest.raises(ValueError):  # the pointwise GEMM is 1x1 ECR only
            sc.ecr_conv_batched(x, f, 1, kernel="Y")


PWSHAPES = [
    # n, c, h, w, k, sparsity: every pointwise tile (401-403), ragged C / K / columns
    (16, 256, 56, 56, 512, 0.7),    # 128 x 128 tiles
    (4, 256, 28, 28, 512, 0.7),
    (3, 13, 9, 11, 200, 0.5),       # C not a multiple of 8, K not of 4, ragged columns
    (2, 480, 14, 14, 192, 0.9),     # GoogLeNet 4a 1x1
    (5, 832, 7, 7, 256, 0.95),
    (1, 1, 1, 1, 1, 0.0),           # one output
    (2, 9, 5, 5, 33, 1.0),          # all zero
]


@pytest.mark.parametrize("shape", PWSHAPES, ids=[str(s) for s in PWSHAPES])
def test_pointwise(sc, orc, shape):
    """1x1 ECR on the dense ordered GEMM: EXACT bit-identical to the oracle
    (zero cells multiplied, not skipped), counters exact, FAST within the bar."""
    n, c, h, w, k, sp = shape
    x, f = inputs(orc, n, c, h, w, k, 1, 1, sp, seed=(hash(shape) ^ 23) & 0xFFFF)
    x[x.view(np.uint32) == 0] = -0.0 if sp < 1 else 0.0  # the reference skips -0 too
    ref, rops = orc.ecr_conv(x, f, 1)
    ops = sc.OpCount()
    assert bits_equal(sc.ecr_conv_batched(x, f, 1, counters=ops, kernel="Y"), ref)
    assert (ops.multiplications, ops.additions) == rops
    assert close(sc.ecr_conv_batched(x, f, 1, fast=True, kernel="Y"), ref)
    assert bits_equal(sc.ecr_conv_batched(x, f, 1), ref)  # default selection


def test_pointwise_nonfinite_weights(sc, orc):
    """An Inf / NaN weight times a zero cell is NaN, which the reference never
    computes (it skips zero cells): the GEMM predicates zero cells off for a
    stage whose weights are not all finite."""
    n, c, h, w, k = 2, 40, 7, 7, 96
    x, f = inputs(orc, n, c, h, w, k, 1, 1, 0.7, seed=404)
    f[3, 17, 0, 0] = np.inf
    f[50, 2, 0, 0] = -np.inf
    f[95, 33, 0, 0] = np.nan
    ref, _ = orc.ecr_conv(x, f, 1)
    for fast in (False, True):
        y = sc.ecr_conv_batched(x, f, 1, fast=fast, kernel="Y")
        nan_ref, nan_y = np.isnan(ref), np.isnan(y)
        assert (nan_ref == nan_y).all()
        if not fast:
            assert bits_equal(np.where(nan_ref, 0, y), np.where(nan_ref, 0, ref))
        else:  # same Inf / NaN positions and values, the finite rest within the bar
            fin = np.isfinite(ref)
            assert (np.isfinite(y) == fin).all() and (y[np.isinf(ref)] == ref[np.isinf(ref)]).all()
            assert close(np.where(fin, y, 0), np.where(fin, ref, 0))


SSHAPES = [
    # n, c, h, w, k, stride, sparsity
    (2, 24, 30, 30, 128, 2, 0.7),
    (2, 16, 31, 29, 160, 2, 0.5),   # ragged tiles, K tail
    (1, 12, 29, 29, 128, 3, 0.7),
    (2, 9, 20, 26, 64, 3, 0.9),
    (1, 8, 17, 17, 256, 2, 0.0),    # dense
]


@pytest.mark.parametrize("shape", SSHAPES, ids=[str(s) for s in SSHAPES])
def test_ws_strided(sc, orc, shape):
    n, c, h, w, k, s, sp = shape
    x, f = inputs(orc, n, c, h, w, k, 3, 3, sp, seed=(hash(shape) ^ 57) & 0xFFFF)
    ref, rops = orc.ecr_conv(x, f, s)
    assert sc.launch_plan(n, c, h, w, k, 3, 3, s)["kernel"] == (111 if s == 2 else 112)
    ops = sc.OpCount()
    assert bits_equal(sc.ecr_conv_batched(x, f, s, counters=ops), ref)
    assert (ops.multiplications, ops.additions) == rops
    assert close(sc.ecr_conv_batched(x, f, s, fast=True), ref)
    assert bits_equal(sc.ecr_conv_batched(x, f, s, kernel="K" if s == 2 else "L"), ref)
    try:
        orc.pack_count(h, 3, s, 2, 2)
        orc.pack_count(w, 3, s, 2, 2)
    except Exception:
        return
    for mode in (0, 1):
        pref, _ = orc.pecr_conv(x, f, s, 2, 2, 2, mode)
        pool = sc.PoolConfig(2, 2, 2, sc.PoolMode(mode))
        assert bits_equal(sc.pecr_conv_pool_batched(x, f, s, pool), pref)
        assert close(sc.pecr_conv_pool_batched(x, f, s, pool, fast=True), pref)


CSHAPES = [
    # n, c, h, w, k, sparsity
    (2, 3, 34, 34, 64, 0.7),     # conv1_1-like
    (3, 1, 19, 23, 96, 0.5),     # ragged tiles, K tail (K-block of 64 half used)
    (1, 4, 18, 18, 128, 0.0),    # dense, two K-blocks
    (2, 2, 10, 14, 32, 1.0),     # all zero
    (2, 3, 66, 34, 128, 0.7),    # 8 tiles per row: shared-memory staged stores, 2 K-blocks
    (1, 3, 35, 66, 64, 0.6),     # staged stores with a partial last tile row
]


@pytest.mark.parametrize("shape", CSHAPES, ids=[str(s) for s in CSHAPES])
def test_smallc(sc, orc, shape):
    n, c, h, w, k, sp = shape
    x, f = inputs(orc, n, c, h, w, k, 3, 3, sp, seed=(hash(shape) ^ 33) & 0xFFFF)
    ref, rops = orc.ecr_conv(x, f, 1)
    # plain ECR: the lanes-over-pixels kernel (301); forced 'M' the per-tile one (300)
    assert sc.launch_plan(n, c, h, w, k, 3, 3, 1)["kernel"] == 301
    ops = sc.OpCount()
    assert bits_equal(sc.ecr_conv_batched(x, f, 1, counters=ops), ref)
    assert (ops.multiplications, ops.additions) == rops
    assert close(sc.ecr_conv_batched(x, f, 1, fast=True), ref)
    assert bits_equal(sc.ecr_conv_batched(x, f, 1, kernel="M"), ref)
    assert close(sc.ecr_conv_batched(x, f, 1, fast=True, kernel="M"), ref)
    if (h - 2) % 2 == 0 and (w - 2) % 2 == 0:
        for mode in (0, 1):
            pref, _ = orc.pecr_conv(x, f, 1, 2, 2, 2, mode)
            pool = sc.PoolConfig(2, 2, 2, sc.PoolMode(mode))
            assert bits_equal(sc.pecr_conv_pool_batched(x, f, 1, pool), pref)
            assert close(sc.pecr_conv_pool_batched(x, f, 1, pool, fast=True), pref)
    # forced on a wider map ('M')
    x2, f2 = inputs(orc, 1, 9, 12, 12, 64, 3, 3, 0.6, seed=5)
    assert bits_equal(sc.ecr_conv_batched(x2, f2, 1, kernel="M"), orc.ecr_conv(x2, f2, 1)[0])


def test_smallc_nonfinite_weights(sc, orc):
    """A zero cell drops out of the sum (ecr_convert keeps only v != 0,
    src/ecr.cpp:84), so an Inf / NaN weight must not reach the outputs whose
    window has a zero there.  The lanes-over-pixels kernel multiplies zero
    cells when every weight is finite and predicates them off otherwise."""
    x, f = inputs(orc, 2, 3, 20, 38, 64, 3, 3, 0.7, seed=91)
    f = f.copy()
    f[3, 1, 1, 1] = np.inf
    f[10, 0, 0, 2] = -np.inf
    f[17, 2, 2, 0] = np.nan
    ref, _ = orc.ecr_conv(x, f, 1)
    for fast in (False, True):
        got = sc.ecr_conv_batched(x, f, 1, fast=fast)
        fin = np.isfinite(ref)
        assert np.array_equal(np.isnan(got), np.isnan(ref))
        assert np.array_equal(got[~fin & ~np.isnan(ref)], ref[~fin & ~np.isnan(ref)])
        if fast:
            assert close(got[fin], ref[fin])
        else:  # NaN payloads may differ between x86 and the GPU; every other value is bit-exact
            nn = ~np.isnan(ref)
            assert bits_equal(got[nn], ref[nn])


@pytest.mark.slow
def test_large_batch_chunking(sc):
    """A device launch whose output exceeds 2^30 elements is cut into image
    chunks (32-bit in-kernel offsets): results equal per-half launches."""
    torch = pytest.importorskip("torch")
    dev = torch.device("cuda:0")
    g = torch.Generator(device=dev)
    g.manual_seed(7)
    # 33 x 64 x 226^2 inputs (108M) -> 33 x 1024 x 224^2 outputs = 1.7e9 elements (6.8 GB)
    x = torch.rand(33, 64, 226, 226, device=dev, generator=g)
    x = x * (torch.rand(x.shape, device=dev, generator=g) >= 0.9)
    w = torch.rand(1024, 64, 3, 3, device=dev, generator=g) - 0.5
    y = sc.ecr_conv_batched(x, w, 1, fast=True)
    for lo, hi in ((0, 1), (16, 17), (32, 33)):
        ref = sc.ecr_conv_batched(x[lo:hi].contiguous(), w, 1, fast=True)
        assert torch.equal(y[lo:hi], ref)
    del y
    torch.cuda.empty_cache()


PSHAPES = [
    # n, c, h, w, k, kh, stride, (pw, ph, ps), sparsity
    (2, 16, 17, 17, 64, 3, 1, (3, 3, 2), 0.7),    # overlapping 3x3/2 (AlexNet-style)
    (1, 24, 14, 20, 128, 3, 1, (2, 3, 1), 0.5),   # non-square, stride 1
    (2, 3, 20, 20, 64, 3, 1, (3, 3, 3), 0.7),     # small C (smallc conv), 3x3/3
    (1, 20, 15, 15, 48, 5, 1, (3, 3, 2), 0.8),    # 5x5 conv, overlapping pool
    (3, 128, 29, 29, 256, 3, 1, (3, 3, 2), 0.7),  # VGG-sized C/K, overlapping pool
    (2, 3, 23, 23, 64, 3, 1, (3, 3, 2), 0.6),     # small C, overlapping pool
    (2, 64, 13, 13, 96, 1, 1, (3, 3, 2), 0.7),    # 1x1 conv (inception), overlapping pool
    (1, 32, 16, 12, 64, 3, 1, (6, 6, 2), 0.7),    # pool as large as the 6x6 conv tile
    (1, 32, 19, 19, 64, 3, 1, (7, 7, 2), 0.7),    # pool larger than any tile: conv + fold
    (2, 16, 23, 23, 64, 3, 2, (3, 3, 2), 0.7),    # strided conv: conv + fold
]


@pytest.mark.parametrize("shape", PSHAPES, ids=[str(s) for s in PSHAPES])
def test_pecr_other_pools(sc, orc, shape):
    """Pools other than 2x2/2, fused: the tile covers whole pool windows and
    the epilogue folds them (one kernel, no pre-pool map in HBM) -- except
    geometries no tile fits, which run conv + pecr_pool_fold_kernel.  Bit-
    identical to the reference's pecr_conv_pool in EXACT mode."""
    n, c, h, w, k, kk, s, (pw, ph, ps), sp = shape
    x, f = inputs(orc, n, c, h, w, k, kk, kk, sp, seed=(hash(shape) ^ 21) & 0xFFFF)
    plan = sc.launch_plan(n, c, h, w, k, kk, kk, s, sc.PoolConfig(pw, ph, ps))
    assert plan["kernel"] != 0
    fused = s == 1 and (pw <= 4 if c <= 4 and kk == 3 else pw <= (6 if kk == 3 else 4))
    ctx = sc.context(0)
    l0 = ctx.launches
    sc.pecr_conv_pool_batched(x, f, s, sc.PoolConfig(pw, ph, ps))
    # filter re-layout + the conv kernel; + pecr_pool_fold_kernel when not fused
    # (whose 3x3 stride-1 conv is a row-prefetch-gated one: + the density
    # gate and the variant not chosen)
    assert ctx.launches - l0 in ((2,) if fused else (3, 5)), plan
    for mode in (0, 1):
        pref, rops = orc.pecr_conv(x, f, s, pw, ph, ps, mode)
        pool = sc.PoolConfig(pw, ph, ps, sc.PoolMode(mode))
        ops = sc.OpCount()
        assert bits_equal(sc.pecr_conv_pool_batched(x, f, s, pool, counters=ops), pref)
        assert (ops.multiplications, ops.additions) == rops
        assert close(sc.pecr_conv_pool_batched(x, f, s, pool, fast=True), pref)


def test_async_host_calls(sc, orc):
    """SCONV_F_ASYNC with host pointers: several layers enqueued back to back
    (rotating workspaces, overlapping transfers) equal the synchronous calls
    once synchronize() returns."""
    torch = pytest.importorskip("torch")
    shapes = [(9, 8, 18, 18, 64, 0), (9, 64, 18, 18, 128, 2), (9, 16, 12, 12, 256, 0),
              (12, 3, 34, 34, 64, 0), (9, 32, 10, 10, 128, 2)]
    xs, ws, want, outs = [], [], [], []
    for i, (n, c, h, w, k, pool) in enumerate(shapes):
        x, f = inputs(orc, n, c, h, w, k, 3, 3, 0.7, seed=300 + i)
        x = torch.from_numpy(x).pin_memory().numpy()
        f = torch.from_numpy(f).pin_memory().numpy()
        if pool:
            ref = sc.pecr_conv_pool_batched(x, f, 1, sc.PoolConfig(2, 2, 2), fast=True)
        else:
            ref = sc.ecr_conv_batched(x, f, 1, fast=True)
        xs.append(x)
        ws.append(f)
        want.append(ref)
        outs.append(torch.empty(ref.shape, dtype=torch.float32).pin_memory().numpy())
    for rep in range(2):
        for (n, c, h, w, k, pool), x, f, o in zip(shapes, xs, ws, outs):
            o.fill(-1.0)
            if pool:
                sc.pecr_conv_pool_batched(x, f, 1, sc.PoolConfig(2, 2, 2), fast=True, out=o,
                                          sync=False)
            else:
                sc.ecr_conv_batched(x, f, 1, fast=True, out=o, sync=False)
        sc.synchronize()
        for o, r in zip(outs, want):
            assert bits_equal(o, r)


def test_sparsity_profiling(sc, orc, ref):
    """window_nnz_counts / sparsity_profile (dataset.cpp:249-286) on the GPU:
    integer window counts equal the oracle's, ratios equal the reference's."""
    maps = []
    for i, (c, h, w, s) in enumerate([(3, 20, 17, 0.7), (3, 20, 17, 0.95), (8, 9, 9, 0.0),
                                      (1, 6, 6, 1.0)]):
        m = orc.generate(h, w, c, s, 70 + i)
        maps.append(sc.FeatureMap(c, h, w, m.reshape(-1)))
    for kk, stride in ((3, 1), (2, 2), (5, 3)):
        for m in maps:
            if kk > min(m.height, m.width):
                continue
            got = sc.window_nnz_counts(m, kk, kk, stride)
            want = orc.window_nnz(m.array(), kk, kk, stride).reshape(-1).tolist()
            assert got == want
        prof = sc.sparsity_profile([m for m in maps if kk <= min(m.height, m.width)], kk, kk,
                                   stride)
        for p, m in zip(prof, [m for m in maps if kk <= min(m.height, m.width)]):
            assert (p.raw, p.extended) == ref.sparsity_profile(m.array(), kk, kk, stride)


@pytest.mark.parametrize("kid", [0, 1, "A", "D", "E", "G", "M", "P", "generic"])
def test_signed_zeros_and_negative_inputs(sc, orc, kid):
    """-0.0 is a zero (`v != 0.0f`, src/ecr.cpp:79-93 / src/pecr.cpp:114-125)
    and negative values are nonzeros: every kernel family must skip the
    former, keep the latter, and give the oracle's bits and counters."""
    c, k = (3, 64) if kid == "M" else (13, 128 if kid in ("A", "E", "P") else 64)
    x, f = inputs(orc, 2, c, 18, 18, k, 3, 3, 0.6, seed=515)
    rng = np.random.default_rng(5)
    zeros = x == 0
    x[zeros & (rng.random(x.shape) < 0.5)] = np.float32(-0.0)
    x[~zeros & (rng.random(x.shape) < 0.3)] *= np.float32(-1.0)
    assert np.signbit(x[zeros]).any() and (x < 0).any()
    generic = kid == "generic"
    kernel = 0 if generic else kid
    ref, rops = orc.ecr_conv(x, f, 1)
    ops = sc.OpCount()
    y = sc.ecr_conv_batched(x, f, 1, counters=ops, generic=generic, kernel=kernel)
    assert bits_equal(y, ref) and (ops.multiplications, ops.additions) == rops
    assert close(sc.ecr_conv_batched(x, f, 1, fast=True, generic=generic, kernel=kernel), ref)
    # the same map with +0.0 everywhere gives the same bits
    xp = np.where(zeros, np.float32(0.0), x).astype(np.float32)
    assert bits_equal(sc.ecr_conv_batched(xp, f, 1, generic=generic, kernel=kernel), y)
    pool = sc.PoolConfig(2, 2, 2)
    pref, pops = orc.pecr_conv(x, f, 1, 2, 2, 2, 0)
    ops = sc.OpCount()
    p = sc.pecr_conv_pool_batched(x, f, 1, pool, counters=ops, generic=generic, kernel=kernel)
    assert bits_equal(p, pref) and (ops.multiplications, ops.additions) == pops


def test_smallc_concurrent_contexts(sc, orc):
    """The small-C kernel keeps each launch's filters in one of 4 constant-memory
    slots per device, copied on the launch's stream and released by an event.
    Six host threads, each with its own context (own stream), run conv1_1-shaped
    launches with different filters at the same time -- more launches in flight
    than slots -- and every output must still be its own filters' result."""
    import ctypes as C
    import threading
    from paper_1909_09927_b200 import _native as nat
    L = nat.lib()
    jobs = []
    for t in range(6):
        x, f = inputs(orc, 3, 3, 34, 66, 64, 3, 3, 0.7, seed=700 + t)
        ref, _ = orc.ecr_conv(x, f, 1)
        jobs.append((np.ascontiguousarray(x), np.ascontiguousarray(f), ref))
    outs = [np.empty_like(j[2]) for j in jobs]
    errs = []

    def work(t):
        try:
            ctx = nat.Context(0)
            x, f, _ = jobs[t]
            for rep in range(4):
                nat.check(L.sconv_cu_ecr_conv(ctx.handle, x.ctypes.data, 3, 3, 34, 66, f.ctypes.data,
                                              64, 3, 3, 1, outs[t].ctypes.data, None, None,
                                              nat.F_EXACT), ctx.handle)
            ctx.close()
        except Exception as e:  # surfaced below
            errs.append(e)

    th = [threading.Thread(target=work, args=(t,)) for t in range(6)]
    for h in th:
        h.start()
    for h in th:
        h.join()
    assert not errs, errs
    for (x, f, ref), got in zip(jobs, outs):
        assert bits_equal(got, ref)
