"""Format export at VGG-19 scale: the reference's two-phase
formats -- ecr_convert's fixed-slot EcrMap (include/sconv/ecr.hpp:35-45) and
pecr_convert's PecrMap (include/sconv/pecr.hpp:39-52) -- produced by the GPU
for full VGG-19 layer inputs (the bench's own generator inputs, image 0,
filter 0), with host pointers (the drop-in's path) and with device pointers
(SCONV_F_DEVICE), against the C oracle array by array: bit-exact.  Then the
second phase (ecr_spmv_conv / pecr_conv_pool) runs over the exported format
and must equal the fused kernels' output for that filter, so the two paths
of the library agree at full size too.

conv1_2's EcrMap is the largest format the reference defines for VGG-19:
224 x 224 windows x 576 slots x 12 bytes = 347 MB per (image, filter).
"""
import ctypes as C

import numpy as np
import pytest

import paper_1909_09927_b200 as sc
from paper_1909_09927_b200 import _native as nat
from paper_1909_09927_b200.workloads import VGG19, vgg_filters, vgg_maps

pytestmark = pytest.mark.gpu

ECR_LAYERS = ["conv1_2", "conv3_1", "conv5_1"]
PECR_LAYERS = ["conv1_2", "conv2_2", "conv4_4", "conv5_4"]


def _layer(name):
    l = [v[0] for v in VGG19].index(name)
    return l, VGG19[l]


def _bits(a):
    return np.ascontiguousarray(a).view(np.uint32)


@pytest.mark.parametrize("name", ECR_LAYERS)
def test_ecr_export_full_size(sc, orc, name):
    l, (_, C_, K, H, _) = _layer(name)
    x = vgg_maps(l, [0], 0.7)[0]
    w = vgg_filters(l, [0])[0]
    ref = orc.ecr_convert(x, w, 1)
    m = sc.FeatureMap(C_, H + 2, H + 2, x)
    f = sc.Filter(C_, 3, 3, w)
    e = sc.ecr_convert(m, f, sc.ConvConfig(1))
    cat = lambda key: np.concatenate([getattr(r, key) for r in e.block_rows])
    assert np.array_equal(cat("ptr"), ref["ptr"].reshape(-1))
    assert np.array_equal(cat("offsets"), ref["offsets"].reshape(-1))
    assert np.array_equal(_bits(cat("f_data")), _bits(ref["f_data"].reshape(-1)))
    assert np.array_equal(_bits(cat("k_data")), _bits(ref["k_data"].reshape(-1)))
    # second phase over the exported format == the fused kernel, bit for bit
    ops = sc.OpCount()
    y = sc.ecr_spmv_conv(e, ops).values.reshape(H, H)
    fops = sc.OpCount()
    yf = sc.ecr_conv_batched(x[None], w[None], 1, counters=fops)[0, 0]
    assert np.array_equal(_bits(y), _bits(yf))
    assert (ops.multiplications, ops.additions) == (fops.multiplications, fops.additions)
    del e, ref


@pytest.mark.parametrize("name", ["conv1_2", "conv5_1"])
def test_ecr_export_device_pointers(sc, orc, name):
    torch = pytest.importorskip("torch")
    l, (_, C_, K, H, _) = _layer(name)
    x = vgg_maps(l, [0], 0.7)[0]
    w = vgg_filters(l, [0])[0]
    ref = orc.ecr_convert(x, w, 1)
    dev = torch.device("cuda:0")
    slot, nwin = C_ * 9, H * H
    xd, wd = torch.from_numpy(x).to(dev), torch.from_numpy(w).to(dev)
    ptr = torch.empty(nwin, dtype=torch.int32, device=dev)
    off = torch.empty(nwin * slot, dtype=torch.int32, device=dev)
    fd = torch.empty(nwin * slot, dtype=torch.float32, device=dev)
    kd = torch.empty(nwin * slot, dtype=torch.float32, device=dev)
    ctx = nat.context(0)
    nat.check(nat.lib().sconv_cu_ecr_convert(ctx.handle, xd.data_ptr(), C_, H + 2, H + 2, wd.data_ptr(),
                                             3, 3, 1, ptr.data_ptr(), off.data_ptr(), fd.data_ptr(),
                                             kd.data_ptr(), nat.F_DEVICE), ctx.handle)
    torch.cuda.synchronize()
    assert np.array_equal(ptr.cpu().numpy(), ref["ptr"].reshape(-1))
    assert np.array_equal(off.cpu().numpy(), ref["offsets"].reshape(-1))
    assert np.array_equal(_bits(fd.cpu().numpy()), _bits(ref["f_data"].reshape(-1)))
    assert np.array_equal(_bits(kd.cpu().numpy()), _bits(ref["k_data"].reshape(-1)))


@pytest.mark.parametrize("name", PECR_LAYERS)
def test_pecr_export_full_size(sc, orc, name):
    l, (_, C_, K, H, _) = _layer(name)
    x = vgg_maps(l, [0], 0.7)[0]
    w = vgg_filters(l, [0])[0]
    ref = orc.pecr_convert(x, 3, 3, 1, 2, 2, 2)
    m = sc.FeatureMap(C_, H + 2, H + 2, x)
    f = sc.Filter(C_, 3, 3, w)
    pool = sc.PoolConfig(2, 2, 2, sc.PoolMode.kMax)
    p = sc.pecr_convert(m, f, sc.ConvConfig(1), pool)
    packs = [pk for row in p.pool_rows for pk in row]
    assert np.array_equal(np.concatenate([pk.count for pk in packs]), ref["count"].reshape(-1))
    assert np.array_equal(np.concatenate([pk.index for pk in packs]), ref["index"])
    assert np.array_equal(_bits(np.concatenate([pk.data for pk in packs])), _bits(ref["data"]))
    ops = sc.OpCount()
    y = sc.pecr_conv_pool(p, ops).values.reshape(H // 2, H // 2)
    fops = sc.OpCount()
    yf = sc.pecr_conv_pool_batched(x[None], w[None], 1, pool, counters=fops)[0, 0]
    assert np.array_equal(_bits(y), _bits(yf))
    assert (ops.multiplications, ops.additions) == (fops.multiplications, fops.additions)


def test_pecr_export_device_pointers(sc, orc):
    torch = pytest.importorskip("torch")
    l, (_, C_, K, H, _) = _layer("conv1_2")
    x = vgg_maps(l, [0], 0.7)[0]
    ref = orc.pecr_convert(x, 3, 3, 1, 2, 2, 2)
    dev = torch.device("cuda:0")
    P = H // 2
    xd = torch.from_numpy(x).to(dev)
    count = torch.empty(P * P * 4, dtype=torch.int32, device=dev)
    start = torch.empty(P * P + 1, dtype=torch.int64, device=dev)
    total = C.c_int64(0)
    ctx = nat.context(0)
    L = nat.lib()
    args = (ctx.handle, xd.data_ptr(), C_, H + 2, H + 2, 3, 3, 1, 2, 2, 2)
    nat.check(L.sconv_cu_pecr_count(*args, count.data_ptr(), start.data_ptr(), C.byref(total),
                                    nat.F_DEVICE), ctx.handle)
    torch.cuda.synchronize()
    t = total.value
    assert t == ref["data"].size
    data = torch.empty(max(t, 1), dtype=torch.float32, device=dev)
    index = torch.empty(max(t, 1), dtype=torch.int32, device=dev)
    nat.check(L.sconv_cu_pecr_fill(*args, start.data_ptr(), t, data.data_ptr(), index.data_ptr(),
                                   nat.F_DEVICE), ctx.handle)
    torch.cuda.synchronize()
    assert np.array_equal(count.cpu().numpy(), ref["count"].reshape(-1))
    assert np.array_equal(start.cpu().numpy(), ref["pack_start"])
    assert np.array_equal(index.cpu().numpy()[:t], ref["index"])
    assert np.array_equal(_bits(data.cpu().numpy()[:t]), _bits(ref["data"]))


def test_pecr_pack_start_scan_many_packs(sc, orc):
    """pack_start is the exclusive prefix of the pack totals (pecr.cpp:126-130,
    kernels/scan.cuh): a 1 x 2898 x 2898 map with 2x2 stride-1 pools has
    2895^2 = 8.4M packs, i.e. more than 1024 scan chunks, so the chunk-offset
    pass runs several 1024-wide tiles with a carry."""
    torch = pytest.importorskip("torch")
    H = 2898
    x = orc.generate(H, H, 1, 0.6, 1234)
    P = (H - 3 + 1 - 2 + 1)  # Eq. 3 with pool stride 1
    dev = torch.device("cuda:0")
    xd = torch.from_numpy(np.ascontiguousarray(x)).to(dev)
    count = torch.empty(P * P * 4, dtype=torch.int32, device=dev)
    start = torch.empty(P * P + 1, dtype=torch.int64, device=dev)
    total = C.c_int64(0)
    ctx = nat.context(0)
    nat.check(nat.lib().sconv_cu_pecr_count(ctx.handle, xd.data_ptr(), 1, H, H, 3, 3, 1, 2, 2, 1,
                                            count.data_ptr(), start.data_ptr(), C.byref(total),
                                            nat.F_DEVICE), ctx.handle)
    torch.cuda.synchronize()
    tot = count.view(-1, 4).sum(1, dtype=torch.int64)
    want = torch.cat([torch.zeros(1, dtype=torch.int64, device=dev), torch.cumsum(tot, 0)])
    assert torch.equal(start, want)
    assert total.value == int(want[-1])
    # the window counts themselves against the oracle's (box sums of nonzeros)
    nnz = orc.window_nnz(x, 3, 3, 1).reshape(H - 2, H - 2)
    c = count.view(P, P, 4).cpu().numpy()
    assert np.array_equal(c[:, :, 0], nnz[:P, :P]) and np.array_equal(c[:, :, 3], nnz[1:P + 1, 1:P + 1])
