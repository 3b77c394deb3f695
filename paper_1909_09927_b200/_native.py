"""ctypes binding of libsconv_cuda.so (include/sconv_cuda.h).

The library is built in-tree by ``paper_1909_09927_b200/csrc/Makefile``
(``__graft_entry__.build()``).  There is no fallback: if the shared object is
missing, importing the compute API raises ImportError, and on a machine
without a B200 every device entry point fails with CudaError.
"""
from __future__ import annotations

import ctypes as C
import os

from .errors import raise_for

HERE = os.path.dirname(os.path.abspath(__file__))
# SCONV_LIB: dev override (A/B of build variants, tools/); the default is the in-tree build
LIB_PATH = os.environ.get("SCONV_LIB") or os.path.join(HERE, "lib", "libsconv_cuda.so")

# exported symbols (kept in sync with include/sconv_cuda.h; tests check both)
SYMBOLS = (
    "sconv_cu_version", "sconv_cu_device_count", "sconv_cu_ctx_create", "sconv_cu_ctx_destroy",
    "sconv_cu_ctx_set_stream", "sconv_cu_ctx_use_own_stream", "sconv_cu_ctx_stream", "sconv_cu_ctx_device",
    "sconv_cu_synchronize", "sconv_cu_last_error", "sconv_cu_launch_count",
    "sconv_conv_output_dims", "sconv_pecr_pack_count", "sconv_cu_plan", "sconv_cu_ecr_conv",
    "sconv_cu_pecr_conv_pool", "sconv_cu_ecr_convert", "sconv_cu_ecr_spmv", "sconv_cu_pecr_count",
    "sconv_cu_pecr_fill", "sconv_cu_pecr_pool", "sconv_shard", "sconv_cu_ecr_conv_multi",
    "sconv_cu_pecr_conv_pool_multi", "sconv_generate", "sconv_generate_batch", "sconv_checksum",
    "sconv_cu_forward", "sconv_cu_forward_dims", "sconv_io_last_error", "sconv_map_file_dims",
    "sconv_load_map", "sconv_save_map", "sconv_load_maps", "sconv_cu_window_nnz",
    "sconv_cu_release_filters", "sconv_packed_dims", "sconv_pack_maps", "sconv_cu_ecr_conv_packed",
    "sconv_cu_pecr_conv_pool_packed", "sconv_cu_unpack_maps",
)

F_EXACT = 0
F_FAST = 1 << 0
F_DEVICE = 1 << 1
F_ASYNC = 1 << 2
F_GENERIC = 1 << 3
F_GRAPH = 1 << 4
F_CACHE_FILTERS = 1 << 5


def F_KERNEL(kid) -> int:
    """SCONV_F_KERNEL: force a tiled configuration (1..6 v2, 'A'..'D' v3)."""
    if isinstance(kid, str):
        kid = ord(kid)
    return (int(kid) & 0xFF) << 8

_vp = C.c_void_p
_i = C.c_int
_u64p = C.POINTER(C.c_uint64)


METHOD_ECR = 1
METHOD_PECR = 2


class LayerDesc(C.Structure):
    """sconv_layer (include/sconv_cuda.h)."""
    _fields_ = [("filters", _vp), ("k", _i), ("kh", _i), ("kw", _i), ("stride", _i), ("relu", _i),
                ("pool_w", _i), ("pool_h", _i), ("pool_stride", _i), ("pool_mode", _i)]


class LaunchPlan(C.Structure):
    _fields_ = [("kernel", _i), ("grid_x", _i), ("grid_y", _i), ("grid_z", _i),
                ("block_threads", _i), ("smem_bytes", _i), ("tile_h", _i), ("tile_w", _i),
                ("tile_k", _i)]


_lib = None


def lib() -> C.CDLL:
    """Load libsconv_cuda.so once; raise ImportError when it was never built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"libsconv_cuda.so not built ({LIB_PATH}); run __graft_entry__.build()")
    L = C.CDLL(LIB_PATH)
    L.sconv_cu_version.restype = C.c_char_p
    L.sconv_cu_device_count.argtypes = [C.POINTER(_i)]
    L.sconv_cu_ctx_create.argtypes = [_i, C.POINTER(_vp)]
    L.sconv_cu_ctx_destroy.argtypes = [_vp]
    L.sconv_cu_ctx_set_stream.argtypes = [_vp, _vp]
    L.sconv_cu_ctx_use_own_stream.argtypes = [_vp]
    L.sconv_cu_ctx_stream.argtypes = [_vp]
    L.sconv_cu_ctx_stream.restype = _vp
    L.sconv_cu_ctx_device.argtypes = [_vp]
    L.sconv_cu_synchronize.argtypes = [_vp]
    L.sconv_cu_last_error.argtypes = [_vp]
    L.sconv_cu_last_error.restype = C.c_char_p
    L.sconv_cu_launch_count.argtypes = [_vp]
    L.sconv_cu_launch_count.restype = C.c_uint64
    L.sconv_cu_release_filters.argtypes = [_vp]
    _i64p = C.POINTER(C.c_int64)
    L.sconv_packed_dims.argtypes = [_i, _i, _i, _i64p, _i64p]
    L.sconv_pack_maps.argtypes = [_vp, _i, _i, _i, _i, _vp, _vp, _vp, C.c_int64, _i64p, _i]
    L.sconv_cu_ecr_conv_packed.argtypes = [_vp, _vp, _vp, _vp] + [_i] * 4 + [_vp] + [_i] * 4 + [
        _vp, _u64p, _u64p, C.c_uint]
    L.sconv_cu_pecr_conv_pool_packed.argtypes = [_vp, _vp, _vp, _vp] + [_i] * 4 + [_vp] + [
        _i] * 8 + [_vp, _u64p, _u64p, C.c_uint]
    L.sconv_cu_unpack_maps.argtypes = [_vp, _vp, _vp, _vp] + [_i] * 4 + [_vp, C.c_uint]
    L.sconv_conv_output_dims.argtypes = [_i] * 5 + [C.POINTER(_i)] * 2
    L.sconv_pecr_pack_count.argtypes = [_i] * 5 + [C.POINTER(_i)]
    L.sconv_cu_plan.argtypes = [_i] * 11 + [C.c_uint, C.POINTER(LaunchPlan)]
    L.sconv_cu_ecr_conv.argtypes = [_vp, _vp] + [_i] * 4 + [_vp] + [_i] * 4 + [_vp, _u64p, _u64p,
                                                                               C.c_uint]
    L.sconv_cu_pecr_conv_pool.argtypes = [_vp, _vp] + [_i] * 4 + [_vp] + [_i] * 8 + [
        _vp, _u64p, _u64p, C.c_uint]
    L.sconv_cu_ecr_convert.argtypes = [_vp, _vp] + [_i] * 3 + [_vp] + [_i] * 3 + [_vp] * 4 + [
        C.c_uint]
    L.sconv_cu_ecr_spmv.argtypes = [_vp, _vp, _vp, _vp] + [_i] * 3 + [_vp, _u64p, _u64p, C.c_uint]
    L.sconv_cu_pecr_count.argtypes = [_vp, _vp] + [_i] * 9 + [_vp, _vp, C.POINTER(C.c_int64),
                                                             C.c_uint]
    L.sconv_cu_pecr_fill.argtypes = [_vp, _vp] + [_i] * 9 + [_vp, C.c_int64, _vp, _vp, C.c_uint]
    L.sconv_cu_pecr_pool.argtypes = [_vp, _vp, _vp, _vp, _vp, C.c_int64, _vp] + [_i] * 8 + [
        _vp, _u64p, _u64p, C.c_uint]
    L.sconv_shard.argtypes = [_i] * 4 + [C.POINTER(_i)] * 4
    L.sconv_cu_ecr_conv_multi.argtypes = [C.POINTER(_vp), _i, _vp] + [_i] * 4 + [_vp] + [
        _i] * 4 + [_vp, _u64p, _u64p, C.c_uint]
    L.sconv_cu_pecr_conv_pool_multi.argtypes = [C.POINTER(_vp), _i, _vp] + [_i] * 4 + [_vp] + [
        _i] * 8 + [_vp, _u64p, _u64p, C.c_uint]
    L.sconv_cu_forward_dims.argtypes = [_vp, _i, _i, _i, _i] + [C.POINTER(_i)] * 3
    L.sconv_cu_forward.argtypes = [_vp, _vp] + [_i] * 4 + [_vp, _i, _i, _vp, _vp, _vp, _u64p,
                                                           _u64p, _vp, C.c_uint]
    L.sconv_cu_window_nnz.argtypes = [_vp, _vp] + [_i] * 7 + [_vp, _vp, _vp, C.c_uint]
    L.sconv_io_last_error.restype = C.c_char_p
    L.sconv_map_file_dims.argtypes = [C.c_char_p] + [C.POINTER(_i)] * 3
    L.sconv_load_map.argtypes = [C.c_char_p, _vp, C.c_int64] + [C.POINTER(_i)] * 3
    L.sconv_save_map.argtypes = [C.c_char_p, _vp, _i, _i, _i]
    L.sconv_load_maps.argtypes = [C.POINTER(C.c_char_p), _i, _vp, _i, _i, _i, _i]
    L.sconv_generate.argtypes = [_i, _i, _i, C.c_double, C.c_uint64, _vp]
    L.sconv_generate_batch.argtypes = [_i, _i, _i, _i, C.c_double, _vp, _vp, _i]
    L.sconv_checksum.argtypes = [_vp, C.c_int64]
    L.sconv_checksum.restype = C.c_uint64
    _lib = L
    return L


def check(status: int, ctx=None) -> None:
    if status:
        msg = lib().sconv_cu_last_error(ctx)
        raise_for(status, msg.decode() if msg else f"status {status}")


class Context:
    """One device + one stream + workspace (sconv_cu_ctx)."""

    def __init__(self, device: int = 0):
        h = _vp()
        check(lib().sconv_cu_ctx_create(device, C.byref(h)))
        self.handle = h
        self.device = device
        self._stream = "own"

    def set_stream(self, stream_ptr: int) -> None:
        """Use an external cudaStream_t (0 = legacy default stream)."""
        if stream_ptr != self._stream:
            check(lib().sconv_cu_ctx_set_stream(self.handle, stream_ptr), self.handle)
            self._stream = stream_ptr

    def use_own_stream(self) -> None:
        if self._stream != "own":
            check(lib().sconv_cu_ctx_use_own_stream(self.handle), self.handle)
            self._stream = "own"

    def synchronize(self) -> None:
        check(lib().sconv_cu_synchronize(self.handle), self.handle)
        self._inflight = []

    def keep(self, *arrays) -> None:
        """Hold host buffers of asynchronous calls until synchronize()."""
        if not hasattr(self, "_inflight"):
            self._inflight = []
        self._inflight.extend(arrays)

    def release_filters(self) -> None:
        """Drop the filter copies kept for cache_filters=True calls."""
        check(lib().sconv_cu_release_filters(self.handle), self.handle)

    @property
    def launches(self) -> int:
        return int(lib().sconv_cu_launch_count(self.handle))

    def close(self) -> None:
        if self.handle:
            lib().sconv_cu_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_contexts: dict[tuple[int, int], Context] = {}


def context(device: int = 0, slot: int = 0) -> Context:
    """The process-wide context `slot` of `device` (slot 0 is the default one;
    further slots are independent contexts on the same device, each with its
    own stream and workspace, e.g. for sconv_cu_*_multi on one GPU)."""
    ctx = _contexts.get((device, slot))
    if ctx is None:
        ctx = _contexts[(device, slot)] = Context(device)
    return ctx
