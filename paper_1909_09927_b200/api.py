"""Python mirror of the reference host API for the ECR / PECR hot path.

Names, argument meaning and error behaviour follow the reference's C++ API
(include/sconv/{tensor,ecr,pecr,exec,metrics,dataset,report}.hpp); every
compute call goes through libsconv_cuda.so (include/sconv_cuda.h) on a B200.
There is no CPU fallback.

Two layers:

* the reference's per-(map, filter) two-phase calls -- ``ecr_convert`` /
  ``ecr_spmv_conv`` / ``pecr_convert`` / ``pecr_conv_pool`` -- which
  materialise the ECR / PECR formats exactly as the reference lays them out
  (bit-exact index, count and value arrays), and
* the batched fused entries -- ``ecr_conv_batched`` and
  ``pecr_conv_pool_batched`` -- that take N maps x K filters (numpy on the
  host, or torch CUDA tensors already in HBM) and never write the format.

``ExecConfig.fast`` selects FFMA arithmetic; the default EXACT mode is
bit-identical to the reference.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import _native as nat
from .errors import ConfigError, FormatError, ShapeError

# ---------------------------------------------------------------------------
# value types (include/sconv/tensor.hpp:12-62, metrics.hpp:11-21)
# ---------------------------------------------------------------------------


def _check_dims(c: int, h: int, w: int, what: str) -> None:
    if c < 1 or h < 1 or w < 1:  # tensor.cpp:11-18
        raise ShapeError(f"{what} dims must be positive, got {c}x{h}x{w}")


@dataclass(eq=False)
class FeatureMap:
    """Dense C x H x W fp32 map; (c, y, x) at c*H*W + y*W + x (tensor.hpp:12-30)."""
    channels: int
    height: int
    width: int
    values: np.ndarray = None

    def __post_init__(self):
        _check_dims(self.channels, self.height, self.width, "feature map")
        n = self.channels * self.height * self.width
        if self.values is None:
            self.values = np.zeros(n, np.float32)
        else:
            self.values = np.ascontiguousarray(self.values, np.float32).reshape(-1)
            if self.values.size != n:
                raise ShapeError("feature map value count does not match dims")

    def size(self) -> int:
        return int(self.values.size)

    def offset(self, c: int, y: int, x: int) -> int:
        return (c * self.height + y) * self.width + x

    def at(self, c: int, y: int, x: int) -> float:
        return float(self.values[self.offset(c, y, x)])

    def array(self) -> np.ndarray:
        return self.values.reshape(self.channels, self.height, self.width)

    def __eq__(self, other):
        return (isinstance(other, FeatureMap) and
                (self.channels, self.height, self.width) ==
                (other.channels, other.height, other.width) and
                np.array_equal(self.values.view(np.uint32), other.values.view(np.uint32)))


@dataclass(eq=False)
class Filter:
    """One convolution kernel, same layout as FeatureMap (tensor.hpp:34-49)."""
    channels: int
    height: int
    width: int
    weights: np.ndarray

    def __post_init__(self):
        _check_dims(self.channels, self.height, self.width, "filter")
        self.weights = np.ascontiguousarray(self.weights, np.float32).reshape(-1)
        if self.weights.size != self.channels * self.height * self.width:
            raise ShapeError("filter weight count does not match dims")

    def size(self) -> int:
        return int(self.weights.size)

    def at(self, c: int, i: int, j: int) -> float:
        return float(self.weights[(c * self.height + i) * self.width + j])

    def array(self) -> np.ndarray:
        return self.weights.reshape(self.channels, self.height, self.width)


@dataclass
class ConvConfig:
    stride: int = 1


class PoolMode(enum.IntEnum):
    kMax = 0
    kMean = 1
    MAX = 0
    MEAN = 1


@dataclass
class PoolConfig:
    width: int = 0
    height: int = 0
    stride: int = 1
    mode: PoolMode = PoolMode.kMax


@dataclass
class ExecConfig:
    """exec.hpp:30-33 plus the device-side knobs.

    ``workers`` keeps the reference's meaning (host worker threads, must be
    >= 1) -- results never depend on it; on the GPU the partition is the CUDA
    grid.  ``device`` picks the B200, ``fast`` selects FFMA arithmetic.
    """
    workers: int = 1
    shared_memory_budget: int = 49152
    device: int = 0
    fast: bool = False


@dataclass
class OpCount:
    multiplications: int = 0
    additions: int = 0

    def merge(self, other: "OpCount") -> None:
        self.multiplications += other.multiplications
        self.additions += other.additions


@dataclass
class OutputDims:
    width: int = 0
    height: int = 0


# ---------------------------------------------------------------------------
# ECR format (include/sconv/ecr.hpp:11-45)
# ---------------------------------------------------------------------------


@dataclass
class EcrDims:
    in_w: int = 0
    in_h: int = 0
    k_w: int = 0
    k_h: int = 0
    stride: int = 1
    channels: int = 1

    def out_w(self) -> int:
        return (self.in_w - self.k_w) // self.stride + 1

    def out_h(self) -> int:
        return (self.in_h - self.k_h) // self.stride + 1

    def slot(self) -> int:
        return self.channels * self.k_w * self.k_h


@dataclass
class EcrBlockRow:
    f_data: np.ndarray
    k_data: np.ndarray
    offsets: np.ndarray
    ptr: np.ndarray


@dataclass
class EcrMap:
    dims: EcrDims
    block_rows: List[EcrBlockRow] = field(default_factory=list)


@dataclass
class EcrGridShape:
    blocks: int = 0
    threads_per_block: int = 0


# ---------------------------------------------------------------------------
# PECR format (include/sconv/pecr.hpp:18-52)
# ---------------------------------------------------------------------------


@dataclass
class PecrDims:
    in_w: int = 0
    in_h: int = 0
    k_w: int = 0
    k_h: int = 0
    conv_stride: int = 1
    channels: int = 1
    pool: PoolConfig = field(default_factory=PoolConfig)

    def tile_w(self) -> int:
        return self.k_w + self.conv_stride * (self.pool.width - 1)

    def tile_h(self) -> int:
        return self.k_h + self.conv_stride * (self.pool.height - 1)

    def windows_per_pack(self) -> int:
        return self.pool.width * self.pool.height

    def capacity(self) -> int:
        return self.windows_per_pack() * self.channels * self.k_w * self.k_h


@dataclass
class PecrPoolPack:
    data: np.ndarray
    index: np.ndarray
    count: np.ndarray


@dataclass
class PecrMap:
    dims: PecrDims
    kernel: np.ndarray
    pool_rows: List[List[PecrPoolPack]] = field(default_factory=list)

    def packs_w(self) -> int:
        return len(self.pool_rows[0]) if self.pool_rows else 0

    def packs_h(self) -> int:
        return len(self.pool_rows)


# ---------------------------------------------------------------------------
# helpers
# ---------------------------------------------------------------------------


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


def _flags(exec_cfg: ExecConfig, extra: int = 0) -> int:
    if exec_cfg.workers < 1:
        raise ConfigError("workers must be >= 1")  # exec.hpp:62
    return (nat.F_FAST if exec_cfg.fast else nat.F_EXACT) | extra


def _ctx(exec_cfg: ExecConfig) -> nat.Context:
    return nat.context(exec_cfg.device)


def conv_output_dims(in_w: int, in_h: int, k_w: int, k_h: int, stride: int) -> OutputDims:
    """tensor.cpp:44-55 (floor semantics, ShapeError / ConfigError)."""
    ow, oh = C.c_int(), C.c_int()
    nat.check(nat.lib().sconv_conv_output_dims(in_w, in_h, k_w, k_h, stride, C.byref(ow),
                                               C.byref(oh)))
    return OutputDims(ow.value, oh.value)


def ecr_grid_shape(in_w: int, in_h: int, k_w: int, k_h: int, stride: int) -> EcrGridShape:
    """(blocks, threads) = (output rows, output cols), ecr.cpp:46-49."""
    d = conv_output_dims(in_w, in_h, k_w, k_h, stride)
    return EcrGridShape(d.height, d.width)


def pecr_pack_count(in_extent: int, k_extent: int, conv_stride: int, pool_extent: int,
                    pool_stride: int) -> int:
    """Eq. 3 with exact-divisibility check, pecr.cpp:62-81."""
    out = C.c_int()
    nat.check(nat.lib().sconv_pecr_pack_count(in_extent, k_extent, conv_stride, pool_extent,
                                              pool_stride, C.byref(out)))
    return out.value


# ---------------------------------------------------------------------------
# ECR two-phase API
# ---------------------------------------------------------------------------


def ecr_convert(map: FeatureMap, filter: Filter, cfg: ConvConfig = ConvConfig(),
                exec: ExecConfig = ExecConfig()) -> EcrMap:
    """ecr_convert (ecr.cpp:51-97) by warp-ballot compaction on the GPU."""
    if filter.channels != map.channels:
        raise ShapeError(f"filter channels {filter.channels} != map channels {map.channels}")
    od = conv_output_dims(map.width, map.height, filter.width, filter.height, cfg.stride)
    dims = EcrDims(map.width, map.height, filter.width, filter.height, cfg.stride, map.channels)
    slot = dims.slot()
    nwin = od.width * od.height
    ptr = np.empty(nwin, np.int32)
    offsets = np.empty(nwin * slot, np.int32)
    f_data = np.empty(nwin * slot, np.float32)
    k_data = np.empty(nwin * slot, np.float32)
    ctx = _ctx(exec)
    nat.check(nat.lib().sconv_cu_ecr_convert(
        ctx.handle, _ptr(map.values), map.channels, map.height, map.width, _ptr(filter.weights),
        filter.height, filter.width, cfg.stride, _ptr(ptr), _ptr(offsets), _ptr(f_data),
        _ptr(k_data), _flags(exec)), ctx.handle)
    rows = []
    row = od.width * slot
    for b in range(od.height):
        rows.append(EcrBlockRow(f_data[b * row:(b + 1) * row], k_data[b * row:(b + 1) * row],
                                offsets[b * row:(b + 1) * row],
                                ptr[b * od.width:(b + 1) * od.width]))
    return EcrMap(dims, rows)


def _check_ecr(ecr: EcrMap) -> None:
    """Structural half of check_ecr (ecr.cpp:22-42); ptr ranges are checked
    by the library."""
    d = ecr.dims
    threads, slot = d.out_w(), d.slot()
    if len(ecr.block_rows) != d.out_h():
        raise FormatError("block row count does not match output height")
    want = threads * slot
    for r in ecr.block_rows:
        if (len(r.f_data) != want or len(r.k_data) != want or len(r.offsets) != want or
                len(r.ptr) != threads):
            raise FormatError("block row arrays do not match thread count")


def ecr_spmv_conv(ecr: EcrMap, counters: Optional[OpCount] = None,
                  exec: ExecConfig = ExecConfig()) -> FeatureMap:
    """ecr_spmv_conv (ecr.cpp:99-128) on the GPU."""
    _check_ecr(ecr)
    d = ecr.dims
    oh, ow, slot = d.out_h(), d.out_w(), d.slot()
    ptr = np.ascontiguousarray(np.concatenate([r.ptr for r in ecr.block_rows]), np.int32)
    f = np.ascontiguousarray(np.concatenate([r.f_data for r in ecr.block_rows]), np.float32)
    k = np.ascontiguousarray(np.concatenate([r.k_data for r in ecr.block_rows]), np.float32)
    out = np.empty(oh * ow, np.float32)
    m, a = C.c_uint64(0), C.c_uint64(0)
    ctx = _ctx(exec)
    nat.check(nat.lib().sconv_cu_ecr_spmv(ctx.handle, _ptr(ptr), _ptr(f), _ptr(k), oh, ow, slot,
                                          _ptr(out), C.byref(m), C.byref(a), _flags(exec)),
              ctx.handle)
    if counters is not None:
        counters.merge(OpCount(m.value, a.value))
    return FeatureMap(1, oh, ow, out)


def ecr_window(ecr: EcrMap, block: int, thread: int) -> np.ndarray:
    """Scatter one window's nonzeros back to a dense slot (ecr.cpp:130-144)."""
    d = ecr.dims
    if block < 0 or block >= d.out_h() or thread < 0 or thread >= d.out_w():
        raise ShapeError("window index out of range")
    row = ecr.block_rows[block]
    slot = d.slot()
    base = thread * slot
    window = np.zeros(slot, np.float32)
    nnz = 0 if row.ptr[thread] == -1 else int(row.ptr[thread])
    window[row.offsets[base:base + nnz]] = row.f_data[base:base + nnz]
    return window


# ---------------------------------------------------------------------------
# PECR two-phase API
# ---------------------------------------------------------------------------


def pecr_convert(map: FeatureMap, filter: Filter, conv: ConvConfig, pool: PoolConfig,
                 exec: ExecConfig = ExecConfig()) -> PecrMap:
    """pecr_convert (pecr.cpp:83-131): count pass, exclusive scan, fill pass."""
    if filter.channels != map.channels:
        raise ShapeError(f"filter channels {filter.channels} != map channels {map.channels}")
    conv_output_dims(map.width, map.height, filter.width, filter.height, conv.stride)
    pw = pecr_pack_count(map.width, filter.width, conv.stride, pool.width, pool.stride)
    ph = pecr_pack_count(map.height, filter.height, conv.stride, pool.height, pool.stride)
    wpp = pool.width * pool.height
    count = np.empty(ph * pw * wpp, np.int32)
    start = np.empty(ph * pw + 1, np.int64)
    total = C.c_int64(0)
    ctx = _ctx(exec)
    L = nat.lib()
    args = (ctx.handle, _ptr(map.values), map.channels, map.height, map.width, filter.height,
            filter.width, conv.stride, pool.width, pool.height, pool.stride)
    nat.check(L.sconv_cu_pecr_count(*args, _ptr(count), _ptr(start), C.byref(total),
                                    _flags(exec)), ctx.handle)
    t = total.value
    data = np.empty(max(t, 1), np.float32)
    index = np.empty(max(t, 1), np.int32)
    nat.check(L.sconv_cu_pecr_fill(*args, _ptr(start), t, _ptr(data), _ptr(index), _flags(exec)),
              ctx.handle)
    dims = PecrDims(map.width, map.height, filter.width, filter.height, conv.stride, map.channels,
                    PoolConfig(pool.width, pool.height, pool.stride, PoolMode(pool.mode)))
    rows = []
    for b in range(ph):
        row = []
        for t_ in range(pw):
            pk = b * pw + t_
            s, e = int(start[pk]), int(start[pk + 1])
            row.append(PecrPoolPack(data[s:e].copy(), index[s:e].copy(),
                                    count[pk * wpp:(pk + 1) * wpp].copy()))
        rows.append(row)
    return PecrMap(dims, filter.weights.copy(), rows)


def pecr_conv_pool(pecr: PecrMap, counters: Optional[OpCount] = None,
                   exec: ExecConfig = ExecConfig()) -> FeatureMap:
    """pecr_conv_pool (pecr.cpp:133-172): fused conv + ReLU + pool over a PecrMap."""
    d = pecr.dims
    packs_w = pecr_pack_count(d.in_w, d.k_w, d.conv_stride, d.pool.width, d.pool.stride)
    packs_h = pecr_pack_count(d.in_h, d.k_h, d.conv_stride, d.pool.height, d.pool.stride)
    if pecr.packs_h() != packs_h:  # check_pecr, pecr.cpp:24-58
        raise FormatError("pack row count mismatch")
    cap = d.channels * d.k_h * d.k_w
    if len(pecr.kernel) != cap:
        raise FormatError("kernel length does not match dims")
    wpp = d.windows_per_pack()
    counts, datas, idxs, start = [], [], [], [0]
    for row in pecr.pool_rows:
        if len(row) != packs_w:
            raise FormatError("pack count mismatch")
        for pack in row:
            if len(pack.count) != wpp:
                raise FormatError("count length does not match windows per pack")
            if len(pack.data) != len(pack.index):
                raise FormatError("data/index length inconsistent with counts")
            counts.append(np.asarray(pack.count, np.int32))
            datas.append(np.asarray(pack.data, np.float32))
            idxs.append(np.asarray(pack.index, np.int32))
            start.append(start[-1] + len(pack.data))
    count = np.ascontiguousarray(np.concatenate(counts), np.int32)
    data = np.ascontiguousarray(np.concatenate(datas + [np.zeros(1, np.float32)]), np.float32)
    index = np.ascontiguousarray(np.concatenate(idxs + [np.zeros(1, np.int32)]), np.int32)
    start = np.asarray(start, np.int64)
    kernel = np.ascontiguousarray(pecr.kernel, np.float32)
    out = np.empty(packs_h * packs_w, np.float32)
    m, a = C.c_uint64(0), C.c_uint64(0)
    ctx = _ctx(exec)
    nat.check(nat.lib().sconv_cu_pecr_pool(
        ctx.handle, _ptr(count), _ptr(start), _ptr(data), _ptr(index), int(start[-1]),
        _ptr(kernel), d.channels, d.k_h, d.k_w, packs_h, packs_w, d.pool.width, d.pool.height,
        int(d.pool.mode), _ptr(out), C.byref(m), C.byref(a), _flags(exec)), ctx.handle)
    if counters is not None:
        counters.merge(OpCount(m.value, a.value))
    return FeatureMap(1, packs_h, packs_w, out)


def pecr_window(pecr: PecrMap, pack_row: int, pack_col: int, n: int) -> np.ndarray:
    """Reconstruct window n of a pack (pecr.cpp:174-189)."""
    d = pecr.dims
    if (pack_row < 0 or pack_row >= pecr.packs_h() or pack_col < 0 or
            pack_col >= pecr.packs_w() or n < 0 or n >= d.windows_per_pack()):
        raise ShapeError("pack window index out of range")
    pack = pecr.pool_rows[pack_row][pack_col]
    pos = int(np.sum(pack.count[:n]))
    window = np.zeros(d.channels * d.k_h * d.k_w, np.float32)
    cn = int(pack.count[n])
    window[pack.index[pos:pos + cn]] = pack.data[pos:pos + cn]
    return window


# ---------------------------------------------------------------------------
# batched fused entries (the hot path)
# ---------------------------------------------------------------------------


def _is_torch_cuda(t) -> bool:
    return hasattr(t, "is_cuda") and bool(getattr(t, "is_cuda"))


def _aligned16(t):
    """The device entries take 16-byte aligned maps (SCONV_F_DEVICE); a view
    at an odd storage offset is copied once instead of faulting."""
    return t if t.data_ptr() % 16 == 0 else t.clone()


@dataclass
class PackedMaps:
    """A batch [n, C, H, W] in the compressed-ingest layout (include/sconv_cuda.h):
    nonzero bitmap `bits` [n, words] (uint32), block offsets `base`
    [n, blocks + 1] (int64, absolute into `values`) and the packed nonzeros
    `values` (float32).  numpy arrays (host; the entries copy exactly these
    bytes) or CUDA tensors (device, see `to`)."""
    shape: tuple
    bits: object
    base: object
    values: object

    @property
    def nbytes(self) -> int:
        """Bytes that cross PCIe for this batch."""
        return int(sum(_nbytes(a) for a in (self.bits, self.base, self.values)))

    def to(self, device) -> "PackedMaps":
        import torch
        t = lambda a: (a if _is_torch_cuda(a) else torch.from_numpy(np.asarray(a))).to(device)
        return PackedMaps(self.shape, t(self.bits), t(self.base), t(self.values))


def _nbytes(a) -> int:
    return a.nbytes if isinstance(a, np.ndarray) else a.numel() * a.element_size()


def pack_maps(x, threads: int = 0) -> PackedMaps:
    """Dense maps [n, C, H, W] (numpy) -> PackedMaps (host, sconv_pack_maps)."""
    x = np.ascontiguousarray(x, np.float32)
    if x.ndim != 4:
        raise ShapeError("pack_maps takes [n, C, H, W]")
    n, c, h, w = x.shape
    L = nat.lib()
    words, blocks = C.c_int64(), C.c_int64()
    nat.check(L.sconv_packed_dims(c, h, w, C.byref(words), C.byref(blocks)))
    nnz = C.c_int64()
    nat.check(L.sconv_pack_maps(_ptr(x), n, c, h, w, None, None, None, 0, C.byref(nnz), threads))
    bits = np.empty((n, words.value), np.uint32)
    base = np.empty((n, blocks.value + 1), np.int64)
    values = np.empty(max(nnz.value, 1), np.float32)
    nat.check(L.sconv_pack_maps(_ptr(x), n, c, h, w, _ptr(bits), _ptr(base), _ptr(values),
                                values.size, C.byref(nnz), threads))
    return PackedMaps((n, c, h, w), bits, base, values[:nnz.value])


def unpack_maps(p: PackedMaps):
    """Expand a device-resident PackedMaps into a dense CUDA tensor
    (sconv_cu_unpack_maps, the kernel the packed entries run before the conv)."""
    import torch
    if not _is_torch_cuda(p.bits):
        raise ShapeError("unpack_maps takes a device PackedMaps (PackedMaps.to)")
    out = torch.empty(p.shape, dtype=torch.float32, device=p.bits.device)
    ctx = nat.context(p.bits.device.index)
    ctx.set_stream(torch.cuda.current_stream(p.bits.device).cuda_stream)
    nat.check(nat.lib().sconv_cu_unpack_maps(ctx.handle, p.bits.data_ptr(), p.base.data_ptr(),
                                             p.values.data_ptr(), *p.shape, out.data_ptr(),
                                             nat.F_DEVICE), ctx.handle)
    return out


def _batched_packed(kind: str, p: PackedMaps, filters, stride: int, pool, mode: int, fast: bool,
                    counters, device: Optional[int], out, sync: bool, flags: int):
    L = nat.lib()
    N, Cc, H, W = p.shape
    dev_in = _is_torch_cuda(p.bits)
    if dev_in:
        import torch
        filters = filters.contiguous()
        dev = p.bits.device.index if device is None else device
        ctx = nat.context(dev)
        ctx.set_stream(torch.cuda.current_stream(p.bits.device).cuda_stream)
        flags |= nat.F_DEVICE
        if not sync and counters is None:
            flags |= nat.F_ASYNC
        ptr = lambda a: a.data_ptr()
    else:
        filters = np.ascontiguousarray(filters, np.float32)
        ctx = nat.context(0 if device is None else device)
        ctx.use_own_stream()
        ptr = _ptr
    K, Cf, kh, kw = filters.shape
    if Cf != Cc:
        raise ShapeError(f"filter channels {Cf} != map channels {Cc}")
    if kind == "ecr":
        od = conv_output_dims(W, H, kw, kh, stride)
        shape = (N, K, od.height, od.width)
    else:
        shape = (N, K, pecr_pack_count(H, kh, stride, pool[1], pool[2]),
                 pecr_pack_count(W, kw, stride, pool[0], pool[2]))
    if out is None:
        if dev_in:
            import torch
            out = torch.empty(shape, dtype=torch.float32, device=p.bits.device)
        else:
            out = np.empty(shape, np.float32)
    elif tuple(out.shape) != shape:
        raise ShapeError("out has the wrong shape")
    if not dev_in and not sync and counters is None:
        flags |= nat.F_ASYNC
        ctx.keep(p.bits, p.base, p.values, filters, out)
    m, a = C.c_uint64(0), C.c_uint64(0)
    mp = C.byref(m) if counters is not None else None
    ap = C.byref(a) if counters is not None else None
    vp = ptr(p.values) if _nbytes(p.values) else None
    if kind == "ecr":
        st = L.sconv_cu_ecr_conv_packed(ctx.handle, ptr(p.bits), ptr(p.base), vp, N, Cc, H, W,
                                        ptr(filters), K, kh, kw, stride, ptr(out), mp, ap, flags)
    else:
        st = L.sconv_cu_pecr_conv_pool_packed(ctx.handle, ptr(p.bits), ptr(p.base), vp, N, Cc, H,
                                              W, ptr(filters), K, kh, kw, stride, pool[0],
                                              pool[1], pool[2], int(mode), ptr(out), mp, ap, flags)
    nat.check(st, ctx.handle)
    if counters is not None:
        counters.merge(OpCount(m.value, a.value))
    return out


def _batched(kind: str, x, filters, stride: int, pool, mode: int, fast: bool, counters,
             device: Optional[int], generic: bool, out, sync: bool, kernel=0,
             cache_filters: bool = False):
    L = nat.lib()
    flags = (nat.F_FAST if fast else 0) | (nat.F_GENERIC if generic else 0)
    if cache_filters:
        flags |= nat.F_CACHE_FILTERS
    if kernel:
        flags |= nat.F_KERNEL(kernel)
    if isinstance(x, PackedMaps):  # compressed ingest
        return _batched_packed(kind, x, filters, stride, pool, mode, fast, counters, device, out,
                               sync, flags)
    if _is_torch_cuda(x):
        import torch
        if not (_is_torch_cuda(filters) and x.dtype == torch.float32 and filters.dtype == torch.float32):
            raise ShapeError("x and filters must both be float32 CUDA tensors")
        dev = x.device.index if device is None else device
        x = _aligned16(x.contiguous())
        filters = filters.contiguous()
        N, Cc, H, W = x.shape
        K, Cf, kh, kw = filters.shape
        if Cf != Cc:
            raise ShapeError(f"filter channels {Cf} != map channels {Cc}")
        if kind == "ecr":
            od = conv_output_dims(W, H, kw, kh, stride)
            shape = (N, K, od.height, od.width)
        else:
            pw = pecr_pack_count(W, kw, stride, pool[0], pool[2])
            ph = pecr_pack_count(H, kh, stride, pool[1], pool[2])
            shape = (N, K, ph, pw)
        user_out = None
        if out is None:
            out = torch.empty(shape, dtype=torch.float32, device=x.device)
        elif tuple(out.shape) != shape or not out.is_contiguous():
            raise ShapeError("out has the wrong shape")
        elif out.data_ptr() % 16:
            user_out, out = out, torch.empty(shape, dtype=torch.float32, device=x.device)
        ctx = nat.context(dev)
        ctx.set_stream(torch.cuda.current_stream(x.device).cuda_stream)
        flags |= nat.F_DEVICE
        if not sync and counters is None:
            flags |= nat.F_ASYNC
        xp, wp, yp = x.data_ptr(), filters.data_ptr(), out.data_ptr()
    else:
        user_out = None
        x = np.ascontiguousarray(x, np.float32)
        filters = np.ascontiguousarray(filters, np.float32)
        N, Cc, H, W = x.shape
        K, Cf, kh, kw = filters.shape
        if Cf != Cc:
            raise ShapeError(f"filter channels {Cf} != map channels {Cc}")
        if kind == "ecr":
            od = conv_output_dims(W, H, kw, kh, stride)
            shape = (N, K, od.height, od.width)
        else:
            pw = pecr_pack_count(W, kw, stride, pool[0], pool[2])
            ph = pecr_pack_count(H, kh, stride, pool[1], pool[2])
            shape = (N, K, ph, pw)
        if out is None:
            out = np.empty(shape, np.float32)
        ctx = nat.context(0 if device is None else device)
        ctx.use_own_stream()
        if not sync and counters is None:
            # asynchronous host-pointer call: the buffers must outlive it
            if not (out.flags.c_contiguous and out.dtype == np.float32):
                raise ShapeError("async calls need a C-contiguous float32 out")
            flags |= nat.F_ASYNC
            ctx.keep(x, filters, out)
        xp, wp, yp = _ptr(x), _ptr(filters), _ptr(out)
    m, a = C.c_uint64(0), C.c_uint64(0)
    mp = C.byref(m) if counters is not None else None
    ap = C.byref(a) if counters is not None else None
    if kind == "ecr":
        st = L.sconv_cu_ecr_conv(ctx.handle, xp, N, Cc, H, W, wp, K, kh, kw, stride, yp, mp, ap,
                                 flags)
    else:
        st = L.sconv_cu_pecr_conv_pool(ctx.handle, xp, N, Cc, H, W, wp, K, kh, kw, stride,
                                       pool[0], pool[1], pool[2], int(mode), yp, mp, ap, flags)
    nat.check(st, ctx.handle)
    if counters is not None:
        counters.merge(OpCount(m.value, a.value))
    if _is_torch_cuda(x) and user_out is not None:
        user_out.copy_(out)
        return user_out
    return out


def synchronize(device: int = 0) -> None:
    """Wait for every call enqueued on `device`'s context (sconv_cu_synchronize);
    host buffers of asynchronous (sync=False) numpy calls are valid after it."""
    nat.context(device).synchronize()


def ecr_conv_batched(x, filters, stride: int = 1, *, fast: bool = False,
                     counters: Optional[OpCount] = None, device: Optional[int] = None,
                     generic: bool = False, out=None, sync: bool = True, kernel=0,
                     cache_filters: bool = False):
    """Fused ECR convolution of x [N,C,H,W] by filters [K,C,kh,kw] -> [N,K,oh,ow].

    Equivalent to multichannel_conv(map, filters, {stride}, Method::kEcr) per
    image (pipeline.cpp:191-210).  numpy in -> numpy out (host copies inside);
    torch CUDA tensors in -> torch out on the current stream.  sync=False
    returns after enqueueing (numpy: pinned buffers overlap; call
    synchronize() before reading out).  `kernel`
    forces a tiled configuration (testing / tuning; SCONV_F_KERNEL).
    `cache_filters` (SCONV_F_CACHE_FILTERS) promises the filter values behind
    this buffer never change: the context keeps their device re-layout.
    """
    return _batched("ecr", x, filters, stride, None, 0, fast, counters, device, generic, out,
                    sync, kernel, cache_filters)


def pecr_conv_pool_batched(x, filters, stride: int = 1, pool: PoolConfig = PoolConfig(2, 2, 2),
                           *, fast: bool = False, counters: Optional[OpCount] = None,
                           device: Optional[int] = None, generic: bool = False, out=None,
                           sync: bool = True, kernel=0, cache_filters: bool = False):
    """Fused conv + ReLU + pooling (forward's fused branch, pipeline.cpp:249-264)."""
    return _batched("pecr", x, filters, stride, (pool.width, pool.height, pool.stride),
                    int(pool.mode), fast, counters, device, generic, out, sync, kernel,
                    cache_filters)


def _multi(kind: str, x, filters, stride: int, pool, mode: int, devices: Sequence[int],
           fast: bool, counters: Optional[OpCount]):
    L = nat.lib()
    x = np.ascontiguousarray(x, np.float32)
    filters = np.ascontiguousarray(filters, np.float32)
    N, Cc, H, W = x.shape
    K, Cf, kh, kw = filters.shape
    if Cf != Cc:
        raise ShapeError(f"filter channels {Cf} != map channels {Cc}")
    if not devices:
        raise ConfigError("no devices")
    # one context per entry: a device listed twice gets two contexts (slots)
    seen: dict[int, int] = {}
    ctxs = []
    for d in devices:
        ctxs.append(nat.context(d, seen.get(d, 0)))
        seen[d] = seen.get(d, 0) + 1
    for c in ctxs:
        c.use_own_stream()
    arr = (C.c_void_p * len(ctxs))(*[c.handle for c in ctxs])
    if kind == "ecr":
        od = conv_output_dims(W, H, kw, kh, stride)
        out = np.empty((N, K, od.height, od.width), np.float32)
    else:
        pw = pecr_pack_count(W, kw, stride, pool[0], pool[2])
        ph = pecr_pack_count(H, kh, stride, pool[1], pool[2])
        out = np.empty((N, K, ph, pw), np.float32)
    m, a = C.c_uint64(0), C.c_uint64(0)
    mp = C.byref(m) if counters is not None else None
    ap = C.byref(a) if counters is not None else None
    flags = nat.F_FAST if fast else 0
    if kind == "ecr":
        st = L.sconv_cu_ecr_conv_multi(arr, len(ctxs), _ptr(x), N, Cc, H, W, _ptr(filters), K, kh,
                                       kw, stride, _ptr(out), mp, ap, flags)
    else:
        st = L.sconv_cu_pecr_conv_pool_multi(arr, len(ctxs), _ptr(x), N, Cc, H, W, _ptr(filters),
                                             K, kh, kw, stride, pool[0], pool[1], pool[2],
                                             int(mode), _ptr(out), mp, ap, flags)
    nat.check(st, None)
    if counters is not None:
        counters.merge(OpCount(m.value, a.value))
    return out


def ecr_conv_multi(x, filters, stride: int = 1, *, devices: Sequence[int] = (0,),
                   fast: bool = False, counters: Optional[OpCount] = None) -> np.ndarray:
    """ECR convolution sharded over several contexts (sconv_cu_ecr_conv_multi):
    each entry of `devices` gets a contiguous shard of the images (or, with
    fewer images than entries, of the filters) -- dispatch over GPUs
    (include/sconv/exec.hpp:57-120).  Host arrays in, host array out."""
    return _multi("ecr", x, filters, stride, None, 0, devices, fast, counters)


def pecr_conv_pool_multi(x, filters, stride: int = 1, pool: PoolConfig = PoolConfig(2, 2, 2), *,
                         devices: Sequence[int] = (0,), fast: bool = False,
                         counters: Optional[OpCount] = None) -> np.ndarray:
    """Fused conv + ReLU + pool sharded over contexts (sconv_cu_pecr_conv_pool_multi)."""
    return _multi("pecr", x, filters, stride, (pool.width, pool.height, pool.stride),
                  int(pool.mode), devices, fast, counters)


def multichannel_conv(map: FeatureMap, filters: Sequence[Filter], cfg: ConvConfig,
                      method: str = "ecr", exec: ExecConfig = ExecConfig(),
                      counters: Optional[OpCount] = None) -> FeatureMap:
    """GPU multichannel_conv (pipeline.cpp:191-210) for Method::kEcr: all K
    filters in one fused launch, output stacked K x oh x ow."""
    if not filters:
        raise ConfigError("multichannel_conv requires filters")
    if method != "ecr":
        raise ConfigError("multichannel_conv on the GPU supports the ecr method only")
    for f in filters:
        if f.channels != map.channels:
            raise ShapeError(f"filter channels {f.channels} != map channels {map.channels}")
        if (f.height, f.width) != (filters[0].height, filters[0].width):
            raise ShapeError("filters must share dims")
    if exec.workers < 1:
        raise ConfigError("workers must be >= 1")
    w = np.stack([f.array() for f in filters])
    y = ecr_conv_batched(map.array()[None], w, cfg.stride, fast=exec.fast, counters=counters,
                         device=exec.device)
    return FeatureMap(len(filters), y.shape[2], y.shape[3], y.reshape(-1))


# ---------------------------------------------------------------------------
# on-device multi-layer forward (include/sconv/pipeline.hpp, src/pipeline.cpp)
# ---------------------------------------------------------------------------


class Activation(enum.IntEnum):
    kNone = 0
    kRelu = 1


class LayerKind(enum.IntEnum):
    kConv = 0
    kConvPool = 1


class Method(enum.IntEnum):
    kDense = 0
    kEcr = 1
    kPecr = 2


@dataclass
class TrafficReport:
    """Modeled byte traffic (include/sconv/metrics.hpp:26-48)."""
    host_to_device_bytes: int = 0
    device_to_host_bytes: int = 0
    global_loads_bytes: int = 0
    global_stores_bytes: int = 0


@dataclass
class LayerSpec:
    """pipeline.hpp:18-24: filters share dims; kConvPool requires `pool`."""
    kind: LayerKind = LayerKind.kConv
    filters: Sequence[Filter] = ()
    conv: ConvConfig = field(default_factory=ConvConfig)
    pool: Optional[PoolConfig] = None
    activation: Activation = Activation.kRelu


@dataclass
class NetworkSpec:
    in_channels: int = 0
    in_height: int = 0
    in_width: int = 0
    layers: List[LayerSpec] = field(default_factory=list)

    def validate(self) -> None:
        """NetworkSpec::validate (pipeline.cpp:154-189)."""
        if self.in_channels < 1 or self.in_height < 1 or self.in_width < 1:
            raise ConfigError("network input dims must be positive")
        if not self.layers:
            raise ConfigError("network has no layers")
        c, h, w = self.in_channels, self.in_height, self.in_width
        for l, layer in enumerate(self.layers):
            where = f"layer {l}: "
            if not layer.filters:
                raise ConfigError(where + "no filters")
            f0 = layer.filters[0]
            for f in layer.filters:
                if (f.channels, f.height, f.width) != (f0.channels, f0.height, f0.width):
                    raise ConfigError(where + "filters have mismatched dims")
            if f0.channels != c:
                raise ConfigError(where + f"filter channels {f0.channels} != input channels {c}")
            if layer.conv.stride < 1:
                raise ConfigError(where + "conv stride must be >= 1")
            if layer.kind == LayerKind.kConvPool and layer.pool is None:
                raise ConfigError(where + "conv_pool layer without pool config")
            if layer.kind == LayerKind.kConv and layer.pool is not None:
                raise ConfigError(where + "conv layer with pool config")
            od = conv_output_dims(w, h, f0.width, f0.height, layer.conv.stride)
            h, w = od.height, od.width
            if layer.pool is not None:
                pd = conv_output_dims(w, h, layer.pool.width, layer.pool.height, layer.pool.stride)
                h, w = pd.height, pd.width
            c = len(layer.filters)


@dataclass
class ForwardResult:
    """pipeline.hpp:37-50."""
    output: FeatureMap
    ops: OpCount = field(default_factory=OpCount)
    traffic: TrafficReport = field(default_factory=TrafficReport)
    conv_outputs: List[FeatureMap] = field(default_factory=list)
    layer_outputs: List[FeatureMap] = field(default_factory=list)
    pecr_fallback_layers: List[int] = field(default_factory=list)


def _layer_descs(layers_w, layer_cfg):
    """(filters [K,C,kh,kw] pointer/array, cfg dict) -> LayerDesc array."""
    arr = (nat.LayerDesc * len(layer_cfg))()
    for l, (wp, cfg) in enumerate(zip(layers_w, layer_cfg)):
        d = arr[l]
        d.filters = wp
        d.k, d.kh, d.kw = cfg["k"], cfg["kh"], cfg["kw"]
        d.stride = cfg["stride"]
        d.relu = int(cfg["relu"])
        pool = cfg.get("pool")
        if pool is not None:
            d.pool_w, d.pool_h, d.pool_stride, d.pool_mode = (pool.width, pool.height, pool.stride,
                                                              int(pool.mode))
    return arr


def forward_batched(x, layers: Sequence[dict], method: Method = Method.kPecr, *,
                    fast: bool = False, counters: Optional[OpCount] = None,
                    device: Optional[int] = None, generic: bool = False,
                    layer_outputs: bool = False, conv_outputs: bool = False, kernel=0,
                    graph: bool = False, out=None):
    """forward() of src/pipeline.cpp:212-301 for a batch x [N,C,H,W] with every
    activation resident on the GPU (sconv_cu_forward).  `layers` is a list of
    dicts {"filters": [K,C,kh,kw], "stride": s, "relu": bool, "pool":
    PoolConfig or None}.  numpy in -> numpy out; torch CUDA in -> torch out.
    `graph` (torch CUDA tensors only): capture the network in a CUDA graph on
    the first call and replay it while x, out and the layers stay the same
    (pass the same `out` tensor each time).  Returns (output, layer_outputs
    list or None, conv_outputs list or None, pecr_fallback_layers)."""
    L = nat.lib()
    if int(method) == Method.kDense:
        raise ConfigError("forward on the GPU runs the compressed methods (ECR, PECR); the dense "
                          "method is the CPU reference's")
    flags = (nat.F_FAST if fast else 0) | (nat.F_GENERIC if generic else 0)
    if kernel:
        flags |= nat.F_KERNEL(kernel)
    if graph:
        flags |= nat.F_GRAPH
    torch_in = _is_torch_cuda(x)
    if torch_in:
        import torch
        x = _aligned16(x.contiguous())
        ws = [lay["filters"].contiguous() for lay in layers]
        dev = x.device.index if device is None else device
        N, Cc, H, W = x.shape
    else:
        x = np.ascontiguousarray(x, np.float32)
        ws = [np.ascontiguousarray(lay["filters"], np.float32) for lay in layers]
        dev = 0 if device is None else device
        N, Cc, H, W = x.shape
    cfg = []
    for lay, w in zip(layers, ws):
        K, Cf, kh, kw = w.shape
        cfg.append({"k": K, "kh": kh, "kw": kw, "stride": lay.get("stride", 1),
                    "relu": lay.get("relu", True), "pool": lay.get("pool")})
    descs = _layer_descs([0] * len(cfg), cfg)
    oc, oh, ow = C.c_int(), C.c_int(), C.c_int()
    nat.check(L.sconv_cu_forward_dims(descs, len(cfg), Cc, H, W, C.byref(oc), C.byref(oh),
                                      C.byref(ow)))
    # per-layer dims (for the optional outputs)
    dims, c, h, w_ = [], Cc, H, W
    for cf in cfg:
        od = conv_output_dims(w_, h, cf["kw"], cf["kh"], cf["stride"])
        pd = od
        if cf["pool"] is not None:
            pd = conv_output_dims(od.width, od.height, cf["pool"].width, cf["pool"].height,
                                  cf["pool"].stride)
        dims.append((cf["k"], od.height, od.width, pd.height, pd.width))
        c, h, w_ = cf["k"], pd.height, pd.width
    if torch_in:
        mk = lambda shape: torch.empty(shape, dtype=torch.float32, device=x.device)
        ptr = lambda t: t.data_ptr()
        ctx = nat.context(dev)
        ctx.set_stream(torch.cuda.current_stream(x.device).cuda_stream)
        flags |= nat.F_DEVICE
    else:
        mk = lambda shape: np.empty(shape, np.float32)
        ptr = _ptr
        ctx = nat.context(dev)
        ctx.use_own_stream()
    descs = _layer_descs([ptr(w) for w in ws], cfg)
    if out is None:
        out = mk((N, oc.value, oh.value, ow.value))
    elif tuple(out.shape) != (N, oc.value, oh.value, ow.value):
        raise ShapeError("out has the wrong shape")
    elif torch_in and out.data_ptr() % 16:
        raise ShapeError("out must be 16-byte aligned (SCONV_F_DEVICE)")
    lo = [mk((N, k, ph, pw)) for k, _, _, ph, pw in dims] if layer_outputs else None
    fused = [int(method) == Method.kPecr and cf["pool"] is not None and cf["relu"] for cf in cfg]
    co = ([None if fz else mk((N, k, h2, w2)) for fz, (k, h2, w2, _, _) in zip(fused, dims)]
          if conv_outputs else None)
    P = C.c_void_p * len(cfg)
    lo_arr = P(*[ptr(t) for t in lo]) if lo else None
    co_arr = P(*[ptr(t) if t is not None else None for t in co]) if co else None
    fb = (C.c_int32 * len(cfg))()
    m, a = C.c_uint64(0), C.c_uint64(0)
    mp = C.byref(m) if counters is not None else None
    ap = C.byref(a) if counters is not None else None
    st = L.sconv_cu_forward(ctx.handle, ptr(x), N, Cc, H, W, descs, len(cfg), int(method),
                            ptr(out), lo_arr, co_arr, mp, ap, fb, flags)
    nat.check(st, ctx.handle)
    if counters is not None:
        counters.merge(OpCount(m.value, a.value))
    return out, lo, co, [l for l in range(len(cfg)) if fb[l]]


def forward(net: NetworkSpec, input: FeatureMap, method: Method,
            exec: ExecConfig = ExecConfig()) -> ForwardResult:
    """GPU forward (pipeline.cpp:212-301): ForwardResult with output, ops,
    per-layer conv/layer outputs, pecr_fallback_layers and the modeled
    traffic of the compressed methods (pipeline.cpp:222-289)."""
    net.validate()
    if (input.channels, input.height, input.width) != (net.in_channels, net.in_height,
                                                        net.in_width):
        raise ShapeError("input dims do not match network spec")
    if exec.workers < 1:
        raise ConfigError("workers must be >= 1")
    layers = [{"filters": np.stack([f.array() for f in lay.filters]), "stride": lay.conv.stride,
               "relu": lay.activation == Activation.kRelu, "pool": lay.pool}
              for lay in net.layers]
    ops = OpCount()
    y, lo, co, fb = forward_batched(input.array()[None], layers, method, fast=exec.fast,
                                    counters=ops, device=exec.device, layer_outputs=True,
                                    conv_outputs=True)
    res = ForwardResult(output=FeatureMap(y.shape[1], y.shape[2], y.shape[3], y.reshape(-1)),
                        ops=ops, pecr_fallback_layers=fb)
    mb = lambda c, h, w: 4 * c * h * w
    t = res.traffic
    t.host_to_device_bytes = mb(input.channels, input.height, input.width) + sum(
        4 * sum(f.size() for f in lay.filters) for lay in net.layers)
    cur = (input.channels, input.height, input.width)
    for l, lay in enumerate(net.layers):
        fbytes = 4 * sum(f.size() for f in lay.filters)
        conv = co[l]
        out = lo[l]
        res.layer_outputs.append(FeatureMap(out.shape[1], out.shape[2], out.shape[3],
                                            out.reshape(-1)))
        t.global_loads_bytes += mb(*cur) + fbytes
        if conv is None:  # fused: the reference stores a 1x1x1 placeholder
            res.conv_outputs.append(FeatureMap(1, 1, 1))
        else:
            res.conv_outputs.append(FeatureMap(conv.shape[1], conv.shape[2], conv.shape[3],
                                               conv.reshape(-1)))
            t.global_stores_bytes += mb(conv.shape[1], conv.shape[2], conv.shape[3])
            if lay.pool is not None:
                t.global_loads_bytes += mb(conv.shape[1], conv.shape[2], conv.shape[3])
        if conv is None or lay.pool is not None:
            t.global_stores_bytes += mb(out.shape[1], out.shape[2], out.shape[3])
        cur = (out.shape[1], out.shape[2], out.shape[3])
    t.device_to_host_bytes = mb(*cur)
    return res


# ---------------------------------------------------------------------------
# datasets / reports / planning
# ---------------------------------------------------------------------------


@dataclass
class SparsityProfile:
    """dataset.hpp:64-67."""
    raw: float = 0.0
    extended: float = 0.0  # zero fraction after im2col extension


def window_nnz_counts(map: FeatureMap, k_w: int, k_h: int, stride: int,
                      device: Optional[int] = None) -> List[int]:
    """window_nnz_counts (dataset.cpp:249-268) on the GPU."""
    od = conv_output_dims(map.width, map.height, k_w, k_h, stride)
    out = np.empty(od.width * od.height, np.int32)
    ctx = nat.context(0 if device is None else device)
    ctx.use_own_stream()
    v = np.ascontiguousarray(map.values, np.float32)
    nat.check(nat.lib().sconv_cu_window_nnz(ctx.handle, _ptr(v), 1, map.channels, map.height,
                                            map.width, k_h, k_w, stride, _ptr(out), None, None,
                                            0), ctx.handle)
    return out.tolist()


def sparsity_profile(maps: Sequence[FeatureMap], k_w: int, k_h: int, stride: int,
                     device: Optional[int] = None) -> List[SparsityProfile]:
    """sparsity_profile (dataset.cpp:270-286) on the GPU: maps of equal dims
    go in one batched call."""
    ctx = nat.context(0 if device is None else device)
    ctx.use_own_stream()
    res = []
    i = 0
    while i < len(maps):
        j = i
        d = (maps[i].channels, maps[i].height, maps[i].width)
        while j < len(maps) and (maps[j].channels, maps[j].height, maps[j].width) == d:
            j += 1
        x = np.stack([np.ascontiguousarray(m.values, np.float32) for m in maps[i:j]])
        raw = np.empty(j - i, np.float64)
        ext = np.empty(j - i, np.float64)
        nat.check(nat.lib().sconv_cu_window_nnz(ctx.handle, _ptr(x), j - i, d[0], d[1], d[2], k_h,
                                                k_w, stride, None, _ptr(raw), _ptr(ext), 0),
                  ctx.handle)
        res.extend(SparsityProfile(float(r), float(e)) for r, e in zip(raw, ext))
        i = j
    return res


def _io_check(st: int) -> None:
    if st:
        from .errors import raise_for
        raise_for(st, nat.lib().sconv_io_last_error().decode())


def load(path) -> FeatureMap:
    """sconv::load (dataset.cpp:240-243): FMAP, or CSV by extension."""
    L = nat.lib()
    c, h, w = C.c_int(), C.c_int(), C.c_int()
    p = str(path).encode()
    _io_check(L.sconv_map_file_dims(p, C.byref(c), C.byref(h), C.byref(w)))
    out = np.empty(c.value * h.value * w.value, np.float32)
    _io_check(L.sconv_load_map(p, _ptr(out), out.size, C.byref(c), C.byref(h), C.byref(w)))
    return FeatureMap(c.value, h.value, w.value, out)


def save(map: FeatureMap, path) -> None:
    """sconv::save (dataset.cpp:232-238)."""
    v = np.ascontiguousarray(map.values, np.float32)
    _io_check(nat.lib().sconv_save_map(str(path).encode(), _ptr(v), map.channels, map.height,
                                       map.width))


def load_batch(paths: Sequence, out=None, threads: int = 0) -> np.ndarray:
    """N same-dims map files -> [N, C, H, W] (into `out`, e.g. a pinned
    buffer, when given), read on host threads (sconv_load_maps)."""
    L = nat.lib()
    if not paths:
        raise ConfigError("no files")
    c, h, w = C.c_int(), C.c_int(), C.c_int()
    _io_check(L.sconv_map_file_dims(str(paths[0]).encode(), C.byref(c), C.byref(h), C.byref(w)))
    shape = (len(paths), c.value, h.value, w.value)
    if out is None:
        out = np.empty(shape, np.float32)
    elif tuple(out.shape) != shape or out.dtype != np.float32 or not out.flags.c_contiguous:
        raise ShapeError("out has the wrong shape")
    arr = (C.c_char_p * len(paths))(*[str(p).encode() for p in paths])
    _io_check(L.sconv_load_maps(arr, len(paths), _ptr(out), c.value, h.value, w.value, threads))
    return out


def generate(height: int, width: int, channels: int, sparsity: float, seed: int) -> FeatureMap:
    """sconv::generate (dataset.cpp:77-100), bit-identical."""
    if not (0.0 <= sparsity <= 1.0):
        raise ConfigError(f"sparsity must be in [0, 1], got {sparsity}")
    _check_dims(channels, height, width, "feature map")
    out = np.empty(channels * height * width, np.float32)
    nat.check(nat.lib().sconv_generate(height, width, channels, float(sparsity), seed, _ptr(out)))
    return FeatureMap(channels, height, width, out)


def generate_batch(seeds: Sequence[int], height: int, width: int, channels: int,
                   sparsity: float, threads: int = 0, out: Optional[np.ndarray] = None) -> np.ndarray:
    """maps[i] = generate(height, width, channels, sparsity, seeds[i]) -> [N,C,H,W]."""
    seeds = np.ascontiguousarray(seeds, np.uint64)
    n = len(seeds)
    if out is None:
        out = np.empty((n, channels, height, width), np.float32)
    nat.check(nat.lib().sconv_generate_batch(n, height, width, channels, float(sparsity),
                                             _ptr(seeds), _ptr(out), threads))
    return out


def checksum_hex(values) -> str:
    """checksum_hex (report.cpp:14-30)."""
    v = np.ascontiguousarray(values, np.float32).reshape(-1)
    return "%016x" % nat.lib().sconv_checksum(_ptr(v), v.size)


def launch_plan(n, c, h, w, k, kh, kw, stride, pool: Optional[PoolConfig] = None,
                fast: bool = False) -> dict:
    p = nat.LaunchPlan()
    pw, ph, ps = (pool.width, pool.height, pool.stride) if pool else (0, 0, 1)
    nat.check(nat.lib().sconv_cu_plan(n, c, h, w, k, kh, kw, stride, pw, ph, ps,
                                      nat.F_FAST if fast else 0, C.byref(p)))
    return {f: getattr(p, f) for f, _ in nat.LaunchPlan._fields_}


def shard(n: int, k: int, world: int, rank: int):
    """sconv_shard: (n_begin, n_end, k_begin, k_end) of `rank`."""
    v = [C.c_int() for _ in range(4)]
    nat.check(nat.lib().sconv_shard(n, k, world, rank, *[C.byref(t) for t in v]))
    return tuple(t.value for t in v)
