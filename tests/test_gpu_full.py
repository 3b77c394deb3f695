"""Full-size parity of every benchmarked configuration, and the host-layer
behaviours that only show on the device (multi-context dispatch, graph
invalidation, filter caching, device-format checks, alignment).

Every VGG-19 layer the bench times (bench.py, paper_1909_09927_b200/workloads.py)
runs at full size on the GPU (N = 2 images of the bench's own inputs, all K
filters) at sparsities 0.5, 0.7 and 0.95, in the mode the bench uses it (ECR,
and PECR conv+ReLU+2x2/2 max pool for the pooled layers, which the sparsity
sweep also times as ECR).  Filters {0, 1, K/2, K-1} of both images are
checked against the C oracle (pinned to the reference by tests/test_oracle.py):
EXACT bit-exact, FAST within |d| <= 1e-5 + 1e-5|ref|.  Where oracle/_ref (the
unmodified reference) is present, filter 0 of image 0 is also checked against
it directly -- the same bar, with no restatement in between.
"""
import ctypes
import os

import numpy as np
import pytest

from paper_1909_09927_b200.workloads import VGG19, vgg_filters, vgg_maps

pytestmark = pytest.mark.gpu

ATOL = 1e-5
RTOL = 1e-5


def bits_equal(a, b):
    a = np.ascontiguousarray(a, np.float32)
    b = np.ascontiguousarray(b, np.float32)
    return a.shape == b.shape and np.array_equal(a.view(np.uint32), b.view(np.uint32))


def close(a, b):
    return bool(np.all(np.abs(a.astype(np.float64) - b) <= ATOL + RTOL * np.abs(b.astype(np.float64))))


CASES = [(l, s) for l in range(len(VGG19)) for s in (0.5, 0.7, 0.95)]


@pytest.fixture(scope="module")
def reflib():
    from oracle.oracle import ref_lib
    return ref_lib()


@pytest.mark.parametrize("case", CASES, ids=[f"{VGG19[l][0]}-s{s}" for l, s in CASES])
def test_vgg_layer_full_size(sc, orc, reflib, case):
    l, s = case
    name, C, K, H, pooled = VGG19[l]
    x = vgg_maps(l, [0, 1], s)
    w = vgg_filters(l)
    ks = [0, 1, K // 2, K - 1]
    pool = sc.PoolConfig(2, 2, 2)
    modes = ["ecr", "pecr"] if pooled else ["ecr"]
    for mode in modes:
        if mode == "pecr":
            ref, rops = orc.pecr_conv(x, w[ks], 1, 2, 2, 2, 0)
        else:
            ref, rops = orc.ecr_conv(x, w[ks], 1)
        for fast in (False, True):
            ops = sc.OpCount()
            if mode == "pecr":
                y = sc.pecr_conv_pool_batched(x, w, 1, pool, fast=fast, counters=ops)
            else:
                y = sc.ecr_conv_batched(x, w, 1, fast=fast, counters=ops)
            got = y[:, ks]
            if fast:
                assert close(got, ref), (name, s, mode)
            else:
                assert bits_equal(got, ref), (name, s, mode)
            # the counters count every filter; the oracle's counted 4 of K
            assert (ops.multiplications * 4, ops.additions * 4) == (rops[0] * K, rops[1] * K)
        if reflib is not None:
            nw = os.cpu_count() or 1
            if mode == "pecr":
                r, _ = reflib.pecr_conv(x[:1], w[:1], 1, 2, 2, 2, 0, workers=nw)
            else:
                r, _ = reflib.ecr_conv(x[:1], w[:1], 1, workers=nw)
            assert bits_equal(r[0, 0], ref[0, 0]), (name, s, mode, "oracle vs reference")


# ---------------------------------------------------------------------------
# multi-context dispatch (sconv_cu_ecr_conv_multi / _pecr_conv_pool_multi):
# two contexts on device 0 stand in for two GPUs -- each has its own stream
# and workspace, exactly as one context per device would.
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("n,k,kind,fast", [(6, 128, "ecr", False), (1, 128, "ecr", False),
                                           (5, 96, "pecr", False), (1, 64, "pecr", True),
                                           (6, 128, "ecr", True), (3, 3, "ecr", False)])
def test_multi_context_dispatch(sc, orc, n, k, kind, fast):
    """Image split (n >= contexts) and output-channel split (n < contexts):
    bit-identical to the single-context call, EXACT bit-identical to the
    oracle, counters summed over the shards (dispatch, exec.hpp:91-118)."""
    x = np.stack([orc.generate(20, 20, 16, 0.7, 400 + i) for i in range(n)])
    w = np.stack([orc.generate(3, 3, 16, 0.0, 500 + j) for j in range(k)]) - np.float32(0.5)
    pool = sc.PoolConfig(2, 2, 2)
    for devs in ([0, 0], [0, 0, 0]):
        ops, ops1 = sc.OpCount(), sc.OpCount()
        if kind == "ecr":
            y = sc.ecr_conv_multi(x, w, 1, devices=devs, fast=fast, counters=ops)
            y1 = sc.ecr_conv_batched(x, w, 1, fast=fast, counters=ops1)
            ref, rops = orc.ecr_conv(x, w, 1)
        else:
            y = sc.pecr_conv_pool_multi(x, w, 1, pool, devices=devs, fast=fast, counters=ops)
            y1 = sc.pecr_conv_pool_batched(x, w, 1, pool, fast=fast, counters=ops1)
            ref, rops = orc.pecr_conv(x, w, 1, 2, 2, 2, 0)
        assert bits_equal(y, y1)
        assert (ops.multiplications, ops.additions) == (ops1.multiplications, ops1.additions) == rops
        if fast:
            assert close(y, ref)
        else:
            assert bits_equal(y, ref)


def test_multi_context_errors(sc):
    L = sc._native.lib()
    assert L.sconv_cu_ecr_conv_multi(None, 0, None, 1, 1, 5, 5, None, 1, 3, 3, 1, None, None,
                                     None, 0) != 0
    arr = (ctypes.c_void_p * 1)(sc.context(0).handle)
    x = np.ones((1, 1, 5, 5), np.float32)
    w = np.ones((1, 1, 3, 3), np.float32)
    y = np.empty((1, 1, 3, 3), np.float32)
    p = lambda a: a.ctypes.data_as(ctypes.c_void_p)
    # device pointers are refused: the multi entry stages host shards itself
    assert L.sconv_cu_ecr_conv_multi(arr, 1, p(x), 1, 1, 5, 5, p(w), 1, 3, 3, 1, p(y), None, None,
                                     sc._native.F_DEVICE) != 0
    with pytest.raises(sc.ShapeError):
        sc.ecr_conv_multi(np.ones((1, 7, 7, 7), np.float32), np.ones((64, 6, 3, 3), np.float32), 1,
                          devices=[0, 0])


# ---------------------------------------------------------------------------
# host-layer behaviours
# ---------------------------------------------------------------------------
def test_graph_replay_after_workspace_growth(sc, orc):
    """A captured forward graph must not replay addresses of a workspace that
    a larger call on the same context has since reallocated."""
    torch = pytest.importorskip("torch")
    dev = torch.device("cuda:0")
    x = torch.from_numpy(np.stack([orc.generate(18, 18, 8, 0.7, 30 + i) for i in range(2)])).to(dev)
    w1 = np.stack([orc.generate(3, 3, 8, 0.0, 60 + j) for j in range(64)]) - np.float32(0.5)
    w2 = np.stack([orc.generate(3, 3, 64, 0.0, 90 + j) for j in range(32)]) - np.float32(0.5)
    layers = [{"filters": torch.from_numpy(w1).to(dev), "stride": 1, "relu": True, "pool": None},
              {"filters": torch.from_numpy(w2).to(dev), "stride": 1, "relu": True,
               "pool": sc.PoolConfig(2, 2, 2)}]
    ref, _, _, _ = sc.forward_batched(x, layers, sc.Method.kPecr)
    out = torch.empty_like(ref)
    sc.forward_batched(x, layers, sc.Method.kPecr, graph=True, out=out)  # eager + capture
    sc.forward_batched(x, layers, sc.Method.kPecr, graph=True, out=out)  # replay
    assert torch.equal(out, ref)
    # a much larger call on the same context grows its workspace (realloc)
    big_x = torch.from_numpy(np.stack([orc.generate(66, 66, 64, 0.7, 7 + i)
                                       for i in range(16)])).to(dev)
    big_w = torch.from_numpy(np.stack([orc.generate(3, 3, 64, 0.0, 8 + j)
                                       for j in range(256)]) - np.float32(0.5)).to(dev)
    sc.ecr_conv_batched(big_x, big_w, 1)
    big_fwd = [dict(layers[0]), dict(layers[1])]
    sc.forward_batched(big_x[:, :8].contiguous(), big_fwd, sc.Method.kPecr)  # grows ctx->fwd
    out.zero_()
    sc.forward_batched(x, layers, sc.Method.kPecr, graph=True, out=out)  # must re-capture
    torch.cuda.synchronize()
    assert torch.equal(out, ref)


def test_cache_filters(sc, orc):
    """SCONV_F_CACHE_FILTERS: the cached re-layout gives the same bits, on
    device and host pointers; a different pointer is a different entry."""
    torch = pytest.importorskip("torch")
    x, w = (np.stack([orc.generate(30, 30, 32, 0.7, 70 + i) for i in range(3)]),
            np.stack([orc.generate(3, 3, 32, 0.0, 80 + j) for j in range(128)]) - np.float32(0.5))
    ref, _ = orc.ecr_conv(x, w, 1)
    for _ in range(3):
        assert bits_equal(sc.ecr_conv_batched(x, w, 1, cache_filters=True), ref)
    xd, wd = torch.from_numpy(x).cuda(), torch.from_numpy(w).cuda()
    for _ in range(3):
        y = sc.ecr_conv_batched(xd, wd, 1, cache_filters=True)
        assert bits_equal(y.cpu().numpy(), ref)
    w2 = w[::-1].copy()
    ref2, _ = orc.ecr_conv(x, w2, 1)
    assert bits_equal(sc.ecr_conv_batched(x, w2, 1, cache_filters=True), ref2)
    p = sc.pecr_conv_pool_batched(xd, wd, 1, sc.PoolConfig(2, 2, 2), cache_filters=True)
    pref, _ = orc.pecr_conv(x, w, 1, 2, 2, 2, 0)
    assert bits_equal(p.cpu().numpy(), pref)
    sc.context(0).release_filters()
    assert bits_equal(sc.ecr_conv_batched(x, w, 1, cache_filters=True), ref)


def test_device_pecr_pool_corrupt_index(sc, orc):
    """A device-resident PECR format with an out-of-range index raises
    FormatError (check_pecr, src/pecr.cpp:24-58) and leaves the context usable."""
    torch = pytest.importorskip("torch")
    L = sc._native.lib()
    m = sc.FeatureMap(2, 8, 8, orc.generate(8, 8, 2, 0.5, 3))
    f = sc.Filter(2, 3, 3, orc.generate(3, 3, 2, 0.0, 4))
    pm = sc.pecr_convert(m, f, sc.ConvConfig(1), sc.PoolConfig(2, 2, 2))
    counts = np.concatenate([p.count for row in pm.pool_rows for p in row]).astype(np.int32)
    data = np.concatenate([p.data for row in pm.pool_rows for p in row]).astype(np.float32)
    index = np.concatenate([p.index for row in pm.pool_rows for p in row]).astype(np.int32)
    starts = np.zeros(len(counts) // 4 + 1, np.int64)
    starts[1:] = np.cumsum(counts.reshape(-1, 4).sum(1))
    index[len(index) // 2] = 1 << 28                       # far outside [0, C*9)
    dc, ds, dd, di = (torch.from_numpy(a).cuda() for a in (counts, starts, data, index))
    dk = torch.from_numpy(np.asarray(f.weights, np.float32)).cuda()
    y = torch.empty(pm.packs_h() * pm.packs_w(), device="cuda")
    ctx = sc.context(0)
    ctx.set_stream(torch.cuda.current_stream().cuda_stream)
    st = L.sconv_cu_pecr_pool(ctx.handle, dc.data_ptr(), ds.data_ptr(), dd.data_ptr(),
                              di.data_ptr(), int(len(index)), dk.data_ptr(), 2, 3, 3,
                              pm.packs_h(), pm.packs_w(), 2, 2, 0, y.data_ptr(), None, None,
                              sc._native.F_DEVICE)
    assert st == 3  # SCONV_ERR_FORMAT
    torch.cuda.synchronize()                               # no sticky fault
    x = np.stack([orc.generate(10, 10, 4, 0.7, 1)])
    w = np.stack([orc.generate(3, 3, 4, 0.0, 2 + j) for j in range(64)]) - np.float32(0.5)
    assert bits_equal(sc.ecr_conv_batched(x, w, 1), orc.ecr_conv(x, w, 1)[0])


def test_misaligned_device_views(sc, orc):
    """A contiguous view at an odd storage offset is not 16-byte aligned: the
    Python layer copies it, the C ABI refuses it (SCONV_ERR_ARG), and no
    kernel faults on a misaligned vector access."""
    torch = pytest.importorskip("torch")
    x = np.stack([orc.generate(18, 18, 8, 0.7, 5 + i) for i in range(2)])
    w = np.stack([orc.generate(3, 3, 8, 0.0, 9 + j) for j in range(64)]) - np.float32(0.5)
    ref, _ = orc.ecr_conv(x, w, 1)
    flat = torch.zeros(x.size + 1, device="cuda")
    flat[1:] = torch.from_numpy(x.reshape(-1)).cuda()
    xv = flat[1:].view(x.shape)
    assert xv.data_ptr() % 16 != 0
    wd = torch.from_numpy(w).cuda()
    assert bits_equal(sc.ecr_conv_batched(xv, wd, 1).cpu().numpy(), ref)
    oflat = torch.empty(ref.size + 1, device="cuda")
    ov = oflat[1:].view(ref.shape)
    sc.ecr_conv_batched(torch.from_numpy(x).cuda(), wd, 1, out=ov)
    assert bits_equal(ov.cpu().numpy(), ref)
    L = sc._native.lib()
    ctx = sc.context(0)
    ctx.set_stream(torch.cuda.current_stream().cuda_stream)
    st = L.sconv_cu_ecr_conv(ctx.handle, xv.data_ptr(), 2, 8, 18, 18, wd.data_ptr(), 64, 3, 3, 1,
                             ov.data_ptr(), None, None, sc._native.F_DEVICE)
    assert st == 7  # SCONV_ERR_ARG


# ---------------------------------------------------------------------------
# compressed ingest: bitmap + packed nonzeros across PCIe, expanded on device
# ---------------------------------------------------------------------------
PACK_SHAPES = [
    # n, c, h, w, k, sparsity, pool
    (3, 16, 22, 22, 128, 0.7, None),
    (5, 64, 30, 30, 64, 0.5, (2, 2, 2)),
    (2, 3, 34, 34, 64, 0.7, None),          # C*H*W not a multiple of 1024
    (4, 32, 17, 17, 64, 0.95, (3, 3, 2)),   # general pool
    (2, 8, 12, 12, 64, 1.0, None),          # all-zero maps
    (21, 128, 16, 16, 256, 0.7, (2, 2, 2)), # several host chunks
]


@pytest.mark.parametrize("shape", PACK_SHAPES, ids=[str(s) for s in PACK_SHAPES])
def test_packed_ingest(sc, orc, shape):
    """The packed entries give the dense entries' bits (EXACT and FAST) and the
    oracle's, with host pointers (the chunked H2D ring) and device pointers."""
    torch = pytest.importorskip("torch")
    n, c, h, w, k, s, pool = shape
    x = np.stack([orc.generate(h, w, c, s, 900 + i) for i in range(n)])
    f = np.stack([orc.generate(3, 3, c, 0.0, 950 + j) for j in range(k)]) - np.float32(0.5)
    p = sc.pack_maps(x)
    assert p.nbytes < x.nbytes or s < 0.05
    pc = None if pool is None else sc.PoolConfig(*pool)
    if pc is None:
        ref, rops = orc.ecr_conv(x, f, 1)
        run = lambda xx, **kw: sc.ecr_conv_batched(xx, f if not kw.pop("dev", False) else fd, 1, **kw)
    else:
        ref, rops = orc.pecr_conv(x, f, 1, *pool, 0)
        run = lambda xx, **kw: sc.pecr_conv_pool_batched(xx, f if not kw.pop("dev", False) else fd,
                                                         1, pc, **kw)
    fd = torch.from_numpy(f).cuda()
    ops = sc.OpCount()
    assert bits_equal(run(p, counters=ops), ref)
    assert (ops.multiplications, ops.additions) == rops
    assert bits_equal(run(p, fast=True), run(x, fast=True))
    pd = p.to("cuda")
    assert bits_equal(run(pd, dev=True).cpu().numpy(), ref)
    xd = sc.unpack_maps(pd)
    expect = np.where(x == 0, np.float32(0), x)   # -0 travels as +0
    assert bits_equal(xd.cpu().numpy(), expect)


def test_packed_async_host_calls(sc, orc):
    """Asynchronous packed host calls back to back (the bench's e2e leg)."""
    xs = [np.stack([orc.generate(18, 18, 32, 0.7, 10 * l + i) for i in range(6)]) for l in range(3)]
    fs = [np.stack([orc.generate(3, 3, 32, 0.0, 500 + 10 * l + j) for j in range(64)]) - np.float32(0.5)
          for l in range(3)]
    ps = [sc.pack_maps(x) for x in xs]
    outs = [np.empty((6, 64, 16, 16), np.float32) for _ in range(3)]
    for _ in range(2):
        for l in range(3):
            sc.ecr_conv_batched(ps[l], fs[l], 1, out=outs[l], sync=False)
        sc.synchronize(0)
        for l in range(3):
            assert bits_equal(outs[l], orc.ecr_conv(xs[l], fs[l], 1)[0])
