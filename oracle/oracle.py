"""ctypes front-end for the parity checkers.  TEST INFRASTRUCTURE ONLY.

Two libraries, both built by ``oracle/Makefile``:

* ``C``   -- ``_build/liboracle.so``, the plain-C restatement of the reference
  hot path (``sconv_oracle.c``; each function cites reference file:line).
* ``Ref`` -- ``_ref/libsconv_ref.so``, the UNMODIFIED reference library
  (``/root/reference/proj/src``) behind a flat C bridge.  Present when it was
  built in the dev container; it travels to the GPU box as a built artefact.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU legs may
import this module.  The product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libsconv_ref.so")

_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_u64p = C.POINTER(C.c_uint64)

STATUS = {1: "ShapeError", 2: "ConfigError", 3: "FormatError", 4: "IoError", 5: "DispatchError"}


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str = ""):
        super().__init__(f"{STATUS.get(code, 'Error')}({code}) {msg}")
        self.code = code
        self.kind = STATUS.get(code, "Error")


def build(ref: bool = True) -> None:
    targets = ["oracle"] + (["ref"] if ref and os.path.isdir("/root/reference/proj") else [])
    subprocess.run(["make", "-s", "-C", HERE] + targets, check=True)


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def out_dims(H, W, kh, kw, stride):
    return (H - kh) // stride + 1, (W - kw) // stride + 1


def pack_dims(H, W, kh, kw, stride, pw, ph, ps):
    def one(i, k, p):
        num = i - k + stride - stride * p + ps * stride
        den = ps * stride
        if num <= 0 or num % den:
            raise OracleError(2, "pool tiling does not divide")
        return num // den
    return one(H, kh, ph), one(W, kw, pw)


class _Lib:
    def __init__(self, path: str):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        self.lib = C.CDLL(path)


class COracle(_Lib):
    """The plain-C restatement (oracle/sconv_oracle.c)."""

    def __init__(self, path: str = ORACLE_SO):
        super().__init__(path)
        L = self.lib
        L.orc_generate.argtypes = [C.c_int, C.c_int, C.c_int, C.c_double, C.c_uint64, _f32p]
        L.orc_dense_conv.argtypes = [_f32p, C.c_int, C.c_int, C.c_int, _f32p, C.c_int, C.c_int,
                                     C.c_int, _f32p, _u64p, _u64p]
        L.orc_pool.argtypes = [_f32p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                               C.c_int, _f32p]
        L.orc_relu.argtypes = [_f32p, C.c_int64, _f32p]
        L.orc_ecr_convert.argtypes = [_f32p, C.c_int, C.c_int, C.c_int, _f32p, C.c_int, C.c_int,
                                      C.c_int, _i32p, _i32p, _f32p, _f32p]
        L.orc_ecr_spmv_conv.argtypes = [_i32p, _f32p, _f32p, C.c_int, C.c_int, C.c_int, _f32p,
                                        _u64p, _u64p]
        L.orc_ecr_conv_batched.argtypes = [_f32p, C.c_int, C.c_int, C.c_int, C.c_int, _f32p,
                                           C.c_int, C.c_int, C.c_int, C.c_int, _f32p, _u64p,
                                           _u64p]
        L.orc_pecr_pack_count.argtypes = [C.c_int] * 5 + [C.POINTER(C.c_int)]
        L.orc_pecr_total.argtypes = [_f32p] + [C.c_int] * 9
        L.orc_pecr_total.restype = C.c_int64
        L.orc_pecr_convert.argtypes = [_f32p] + [C.c_int] * 9 + [_i32p, _i64p, _f32p, _i32p]
        L.orc_pecr_conv_pool.argtypes = [_i32p, _i64p, _f32p, _i32p, _f32p] + [C.c_int] * 8 + [
            _f32p, _u64p, _u64p]
        L.orc_pecr_conv_pool_batched.argtypes = [_f32p, C.c_int, C.c_int, C.c_int, C.c_int,
                                                 _f32p] + [C.c_int] * 8 + [_f32p, _u64p, _u64p]
        L.orc_window_nnz.argtypes = [_f32p] + [C.c_int] * 6 + [_i32p]
        L.orc_checksum.argtypes = [_f32p, C.c_int64]
        L.orc_checksum.restype = C.c_uint64
        L.orc_rng_seed.argtypes = [C.c_void_p, C.c_uint64]
        L.orc_rng_next.argtypes = [C.c_void_p]
        L.orc_rng_next.restype = C.c_uint64

    @staticmethod
    def _chk(rc):
        if rc:
            raise OracleError(rc)

    def rng(self, seed: int, n: int):
        st = (C.c_uint64 * 4)()
        self.lib.orc_rng_seed(C.byref(st), seed)
        return [self.lib.orc_rng_next(C.byref(st)) for _ in range(n)]

    def generate(self, h, w, c, sparsity, seed):
        out = np.empty(c * h * w, np.float32)
        self._chk(self.lib.orc_generate(h, w, c, sparsity, seed, out))
        return out.reshape(c, h, w)

    def dense_conv(self, x, w, stride):
        x, w = _f32(x), _f32(w)
        Cc, H, W = x.shape
        _, kh, kw = w.shape
        oh, ow = out_dims(H, W, kh, kw, stride)
        y = np.empty(max(oh, 0) * max(ow, 0), np.float32)
        m, a = C.c_uint64(0), C.c_uint64(0)
        self._chk(self.lib.orc_dense_conv(x, Cc, H, W, w, kh, kw, stride, y, C.byref(m), C.byref(a)))
        return y.reshape(oh, ow), (m.value, a.value)

    def relu(self, x):
        x = _f32(x)
        y = np.empty_like(x)
        self.lib.orc_relu(x.reshape(-1), x.size, y.reshape(-1))
        return y

    def pool(self, x, pw, ph, ps, mode=0):
        x = _f32(x)
        Cc, H, W = x.shape
        oh, ow = out_dims(H, W, ph, pw, ps)
        y = np.empty(Cc * oh * ow, np.float32)
        self._chk(self.lib.orc_pool(x, Cc, H, W, pw, ph, ps, mode, y))
        return y.reshape(Cc, oh, ow)

    def ecr_convert(self, x, w, stride):
        x, w = _f32(x), _f32(w)
        Cc, H, W = x.shape
        _, kh, kw = w.shape
        oh, ow = out_dims(H, W, kh, kw, stride)
        slot = Cc * kh * kw
        ptr = np.empty(oh * ow, np.int32)
        off = np.empty(oh * ow * slot, np.int32)
        fd = np.empty(oh * ow * slot, np.float32)
        kd = np.empty(oh * ow * slot, np.float32)
        self._chk(self.lib.orc_ecr_convert(x, Cc, H, W, w, kh, kw, stride, ptr, off, fd, kd))
        return dict(ptr=ptr.reshape(oh, ow), offsets=off.reshape(oh, ow, slot),
                    f_data=fd.reshape(oh, ow, slot), k_data=kd.reshape(oh, ow, slot))

    def ecr_spmv(self, ptr, f_data, k_data):
        ptr = np.ascontiguousarray(ptr, np.int32)
        oh, ow, slot = f_data.shape
        y = np.empty(oh * ow, np.float32)
        m, a = C.c_uint64(0), C.c_uint64(0)
        self._chk(self.lib.orc_ecr_spmv_conv(ptr.reshape(-1), _f32(f_data).reshape(-1),
                                             _f32(k_data).reshape(-1), oh, ow, slot, y,
                                             C.byref(m), C.byref(a)))
        return y.reshape(oh, ow), (m.value, a.value)

    def ecr_conv(self, x, w, stride):
        """x [N,C,H,W], w [K,C,kh,kw] -> y [N,K,oh,ow], (muls, adds)."""
        x, w = _f32(x), _f32(w)
        N, Cc, H, W = x.shape
        K, _, kh, kw = w.shape
        oh, ow = out_dims(H, W, kh, kw, stride)
        y = np.empty(N * K * oh * ow, np.float32)
        m, a = C.c_uint64(0), C.c_uint64(0)
        self._chk(self.lib.orc_ecr_conv_batched(x.reshape(-1), N, Cc, H, W, w.reshape(-1), K, kh,
                                                kw, stride, y, C.byref(m), C.byref(a)))
        return y.reshape(N, K, oh, ow), (m.value, a.value)

    def pack_count(self, i, k, cs, p, ps):
        out = C.c_int(0)
        self._chk(self.lib.orc_pecr_pack_count(i, k, cs, p, ps, C.byref(out)))
        return out.value

    def pecr_convert(self, x, kh, kw, stride, pw, ph, ps):
        x = _f32(x)
        Cc, H, W = x.shape
        pH, pW = pack_dims(H, W, kh, kw, stride, pw, ph, ps)
        total = self.lib.orc_pecr_total(x, Cc, H, W, kh, kw, stride, pw, ph, ps)
        if total < 0:
            raise OracleError(int(-total))
        count = np.empty(pH * pW * pw * ph, np.int32)
        start = np.empty(pH * pW + 1, np.int64)
        data = np.empty(max(total, 1), np.float32)
        index = np.empty(max(total, 1), np.int32)
        self._chk(self.lib.orc_pecr_convert(x, Cc, H, W, kh, kw, stride, pw, ph, ps, count, start,
                                            data, index))
        return dict(count=count.reshape(pH, pW, pw * ph), pack_start=start,
                    data=data[:total], index=index[:total])

    def pecr_conv_pool(self, fmt, kernel, pw, ph, mode=0):
        kernel = _f32(kernel)
        Cc, kh, kw = kernel.shape
        pH, pW, _ = fmt["count"].shape
        y = np.empty(pH * pW, np.float32)
        m, a = C.c_uint64(0), C.c_uint64(0)
        data = np.ascontiguousarray(fmt["data"], np.float32)
        index = np.ascontiguousarray(fmt["index"], np.int32)
        if data.size == 0:
            data, index = np.zeros(1, np.float32), np.zeros(1, np.int32)
        self._chk(self.lib.orc_pecr_conv_pool(
            np.ascontiguousarray(fmt["count"], np.int32).reshape(-1),
            np.ascontiguousarray(fmt["pack_start"], np.int64), data, index,
            kernel.reshape(-1), Cc, kh, kw, pH, pW, pw, ph, mode, y, C.byref(m), C.byref(a)))
        return y.reshape(pH, pW), (m.value, a.value)

    def pecr_conv(self, x, w, stride, pw, ph, ps, mode=0):
        """x [N,C,H,W], w [K,C,kh,kw] -> pooled y [N,K,pH,pW], (muls, adds)."""
        x, w = _f32(x), _f32(w)
        N, Cc, H, W = x.shape
        K, _, kh, kw = w.shape
        pH, pW = pack_dims(H, W, kh, kw, stride, pw, ph, ps)
        y = np.empty(N * K * pH * pW, np.float32)
        m, a = C.c_uint64(0), C.c_uint64(0)
        self._chk(self.lib.orc_pecr_conv_pool_batched(x.reshape(-1), N, Cc, H, W, w.reshape(-1), K,
                                                      kh, kw, stride, pw, ph, ps, mode, y,
                                                      C.byref(m), C.byref(a)))
        return y.reshape(N, K, pH, pW), (m.value, a.value)

    def window_nnz(self, x, kh, kw, stride):
        x = _f32(x)
        Cc, H, W = x.shape
        oh, ow = out_dims(H, W, kh, kw, stride)
        out = np.empty(oh * ow, np.int32)
        self._chk(self.lib.orc_window_nnz(x, Cc, H, W, kh, kw, stride, out))
        return out.reshape(oh, ow)

    def checksum(self, v) -> str:
        v = _f32(v).reshape(-1)
        return "%016x" % self.lib.orc_checksum(v, v.size)

    def forward(self, x, layers, method):
        """forward() of src/pipeline.cpp:212-301 for one image x [C,H,W],
        composed from this oracle's restated primitives.  `layers`: dicts
        {"filters": [K,C,kh,kw], "stride", "relu", "pool": (pw, ph, ps, mode)
        or None}; method 0 dense / 1 ECR / 2 PECR.  Returns (output,
        layer_outputs, conv_outputs, (muls, adds), pecr_fallback_layers);
        conv_outputs[l] is None where the reference stores its 1x1x1
        placeholder (fused layers, pipeline.cpp:258)."""
        cur = _f32(x)
        lo, co, fb = [], [], []
        m = a = 0
        for l, lay in enumerate(layers):
            w = _f32(lay["filters"])
            s = lay.get("stride", 1)
            relu = lay.get("relu", True)
            pool = lay.get("pool")
            fuse = method == 2 and pool is not None and relu          # :238-240
            if fuse:                                                   # :249-264
                y, (dm, da) = self.pecr_conv(cur[None], w, s, pool[0], pool[1], pool[2], pool[3])
                co.append(None)
                cur = y[0]
            else:
                if method == 2:
                    fb.append(l)                                       # :266-268
                if method == 0:                                        # :241-248
                    outs = [self.dense_conv(cur, w[k], s) for k in range(w.shape[0])]
                    conv = np.stack([o[0] for o in outs])
                    dm, da = sum(o[1][0] for o in outs), sum(o[1][1] for o in outs)
                else:                                                  # :269-285
                    y, (dm, da) = self.ecr_conv(cur[None], w, s)
                    conv = y[0]
                co.append(conv)
                cur = self.relu(conv) if relu else conv
                if pool is not None:
                    cur = self.pool(cur, pool[0], pool[1], pool[2], pool[3])
            m += dm
            a += da
            lo.append(cur)
        return cur, lo, co, (m, a), fb


class RefLib(_Lib):
    """The unmodified reference library through oracle/ref_bridge.cpp."""

    def __init__(self, path: str = REF_SO):
        super().__init__(path)
        L = self.lib
        L.ref_last_error.restype = C.c_char_p
        L.ref_rng.argtypes = [C.c_uint64, C.c_int, np.ctypeslib.ndpointer(np.uint64)]
        L.ref_generate.argtypes = [C.c_int, C.c_int, C.c_int, C.c_double, C.c_uint64, _f32p]
        L.ref_fixture_f5.argtypes = [_f32p]
        L.ref_fixture_k3.argtypes = [_f32p]
        L.ref_dense_conv.argtypes = [_f32p, C.c_int, C.c_int, C.c_int, _f32p, C.c_int, C.c_int,
                                     C.c_int, _f32p, _u64p, _u64p]
        L.ref_relu_pool.argtypes = [_f32p] + [C.c_int] * 8 + [_f32p]
        L.ref_ecr_convert.argtypes = [_f32p, C.c_int, C.c_int, C.c_int, _f32p] + [C.c_int] * 4 + [
            _i32p, _i32p, _f32p, _f32p]
        L.ref_ecr_conv.argtypes = [_f32p, C.c_int, C.c_int, C.c_int, C.c_int, _f32p] + [
            C.c_int] * 5 + [_f32p, _u64p, _u64p]
        L.ref_pecr_pack_count.argtypes = [C.c_int] * 5 + [C.POINTER(C.c_int)]
        L.ref_pecr_convert.argtypes = [_f32p, C.c_int, C.c_int, C.c_int, _f32p] + [C.c_int] * 7 + [
            C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(C.c_int64)]
        L.ref_pecr_conv.argtypes = [_f32p, C.c_int, C.c_int, C.c_int, C.c_int, _f32p] + [
            C.c_int] * 9 + [_f32p, _u64p, _u64p]
        L.ref_window_nnz.argtypes = [_f32p] + [C.c_int] * 6 + [_i32p]
        L.ref_checksum.argtypes = [_f32p, C.c_int64, C.c_char_p]
        L.ref_plan.argtypes = [C.c_int] * 10 + [C.POINTER(C.c_int), C.POINTER(C.c_int), _u64p]
        L.ref_hardware_concurrency.restype = C.c_int
        L.ref_sparsity_profile.argtypes = [_f32p] + [C.c_int] * 6 + [C.POINTER(C.c_double)] * 2
        L.ref_save_map.argtypes = [C.c_char_p, _f32p, C.c_int, C.c_int, C.c_int]
        L.ref_load_map.argtypes = [C.c_char_p, _f32p, C.c_int64] + [C.POINTER(C.c_int)] * 3
        L.ref_forward.argtypes = [_f32p] + [C.c_int] * 4 + [C.c_void_p] * 10 + [C.c_int, C.c_int,
                                  _f32p, _f32p, _u64p, _u64p, C.c_void_p]

    def _chk(self, rc):
        if rc:
            raise OracleError(rc, self.lib.ref_last_error().decode())

    def hardware_concurrency(self):
        return self.lib.ref_hardware_concurrency()

    def sparsity_profile(self, x, kw, kh, stride):
        x = _f32(x)
        raw, ext = C.c_double(), C.c_double()
        self._chk(self.lib.ref_sparsity_profile(x.reshape(-1), *x.shape, kw, kh, stride,
                                                C.byref(raw), C.byref(ext)))
        return raw.value, ext.value

    def save_map(self, x, path):
        x = _f32(x)
        self._chk(self.lib.ref_save_map(str(path).encode(), x.reshape(-1), *x.shape))

    def load_map(self, path, cap=1 << 24):
        out = np.empty(cap, np.float32)
        c, h, w = C.c_int(), C.c_int(), C.c_int()
        self._chk(self.lib.ref_load_map(str(path).encode(), out, cap, C.byref(c), C.byref(h),
                                        C.byref(w)))
        return out[:c.value * h.value * w.value].reshape(c.value, h.value, w.value)

    def forward(self, x, layers, method, workers=1):
        """sconv::forward (pipeline.cpp:212-301) of the unmodified reference on
        one image; same return shape as COracle.forward."""
        x = _f32(x)
        Cc, H, W = x.shape
        nl = len(layers)
        I = C.c_int * nl
        ks, khs, kws, ss, rl = I(), I(), I(), I(), I()
        pws, phs, pss, pms = I(), I(), I(), I()
        fl = (C.c_void_p * nl)()
        keep = []
        sizes, csizes = [], []
        h, w_ = H, W
        for l, lay in enumerate(layers):
            f = _f32(lay["filters"])
            keep.append(f)
            K, _, kh, kw = f.shape
            s = lay.get("stride", 1)
            ks[l], khs[l], kws[l], ss[l], rl[l] = K, kh, kw, s, int(lay.get("relu", True))
            pool = lay.get("pool")
            oh, ow = out_dims(h, w_, kh, kw, s)
            csizes.append((K, oh, ow))
            if pool is not None:
                pws[l], phs[l], pss[l], pms[l] = pool
                oh, ow = out_dims(oh, ow, pool[1], pool[0], pool[2])
            fl[l] = f.ctypes.data
            sizes.append((K, oh, ow))
            h, w_ = oh, ow
        lo_buf = np.zeros(sum(k * a * b for k, a, b in sizes), np.float32)
        co_buf = np.zeros(sum(k * a * b for k, a, b in csizes), np.float32)
        m, a = C.c_uint64(0), C.c_uint64(0)
        fb = (C.c_int * nl)()
        self._chk(self.lib.ref_forward(x.reshape(-1), Cc, H, W, nl, ks, khs, kws, ss, rl, pws, phs,
                                       pss, pms, fl, method, workers, lo_buf, co_buf, C.byref(m),
                                       C.byref(a), fb))
        lo, co, p, q = [], [], 0, 0
        for l, ((k, oh, ow), (ck, ch, cw)) in enumerate(zip(sizes, csizes)):
            lo.append(lo_buf[p:p + k * oh * ow].reshape(k, oh, ow))
            p += k * oh * ow
            fused = method == 2 and layers[l].get("pool") is not None and layers[l].get("relu", True)
            co.append(None if fused else co_buf[q:q + ck * ch * cw].reshape(ck, ch, cw))
            q += ck * ch * cw
        return lo[-1], lo, co, (m.value, a.value), [l for l in range(nl) if fb[l]]

    def rng(self, seed, n):
        out = np.empty(n, np.uint64)
        self.lib.ref_rng(seed, n, out)
        return [int(v) for v in out]

    def generate(self, h, w, c, sparsity, seed):
        out = np.empty(c * h * w, np.float32)
        self._chk(self.lib.ref_generate(h, w, c, sparsity, seed, out))
        return out.reshape(c, h, w)

    def fixtures(self):
        f5 = np.empty(25, np.float32)
        k3 = np.empty(9, np.float32)
        self.lib.ref_fixture_f5(f5)
        self.lib.ref_fixture_k3(k3)
        return f5.reshape(1, 5, 5), k3.reshape(1, 3, 3)

    def dense_conv(self, x, w, stride):
        x, w = _f32(x), _f32(w)
        Cc, H, W = x.shape
        _, kh, kw = w.shape
        oh, ow = out_dims(H, W, kh, kw, stride)
        y = np.empty(max(oh * ow, 1), np.float32)
        m, a = C.c_uint64(0), C.c_uint64(0)
        self._chk(self.lib.ref_dense_conv(x, Cc, H, W, w, kh, kw, stride, y, C.byref(m), C.byref(a)))
        return y[:oh * ow].reshape(oh, ow), (m.value, a.value)

    def relu_pool(self, x, pw, ph, ps, mode=0, relu_first=True):
        x = _f32(x)
        Cc, H, W = x.shape
        oh, ow = out_dims(H, W, ph, pw, ps)
        y = np.empty(max(Cc * oh * ow, 1), np.float32)
        self._chk(self.lib.ref_relu_pool(x, Cc, H, W, int(relu_first), pw, ph, ps, mode, y))
        return y[:Cc * oh * ow].reshape(Cc, oh, ow)

    def ecr_convert(self, x, w, stride, workers=1):
        x, w = _f32(x), _f32(w)
        Cc, H, W = x.shape
        _, kh, kw = w.shape
        oh, ow = out_dims(H, W, kh, kw, stride)
        slot = Cc * kh * kw
        ptr = np.empty(max(oh * ow, 1), np.int32)
        off = np.empty(max(oh * ow * slot, 1), np.int32)
        fd = np.empty(max(oh * ow * slot, 1), np.float32)
        kd = np.empty(max(oh * ow * slot, 1), np.float32)
        self._chk(self.lib.ref_ecr_convert(x, Cc, H, W, w, kh, kw, stride, workers, ptr, off, fd, kd))
        n = oh * ow
        return dict(ptr=ptr[:n].reshape(oh, ow), offsets=off[:n * slot].reshape(oh, ow, slot),
                    f_data=fd[:n * slot].reshape(oh, ow, slot),
                    k_data=kd[:n * slot].reshape(oh, ow, slot))

    def ecr_conv(self, x, w, stride, workers=1):
        x, w = _f32(x), _f32(w)
        N, Cc, H, W = x.shape
        K, _, kh, kw = w.shape
        oh, ow = out_dims(H, W, kh, kw, stride)
        y = np.empty(N * K * oh * ow, np.float32)
        m, a = C.c_uint64(0), C.c_uint64(0)
        self._chk(self.lib.ref_ecr_conv(x.reshape(-1), N, Cc, H, W, w.reshape(-1), K, kh, kw,
                                        stride, workers, y, C.byref(m), C.byref(a)))
        return y.reshape(N, K, oh, ow), (m.value, a.value)

    def pack_count(self, i, k, cs, p, ps):
        out = C.c_int(0)
        self._chk(self.lib.ref_pecr_pack_count(i, k, cs, p, ps, C.byref(out)))
        return out.value

    def pecr_convert(self, x, w, stride, pw, ph, ps, workers=1):
        x, w = _f32(x), _f32(w)
        Cc, H, W = x.shape
        _, kh, kw = w.shape
        total = C.c_int64(0)
        self._chk(self.lib.ref_pecr_convert(x, Cc, H, W, w, kh, kw, stride, pw, ph, ps, workers,
                                            None, None, None, None, C.byref(total)))
        pH, pW = pack_dims(H, W, kh, kw, stride, pw, ph, ps)
        t = total.value
        count = np.empty(pH * pW * pw * ph, np.int32)
        start = np.empty(pH * pW + 1, np.int64)
        data = np.empty(max(t, 1), np.float32)
        index = np.empty(max(t, 1), np.int32)
        self._chk(self.lib.ref_pecr_convert(x, Cc, H, W, w, kh, kw, stride, pw, ph, ps, workers,
                                            count.ctypes.data, start.ctypes.data, data.ctypes.data,
                                            index.ctypes.data, C.byref(total)))
        return dict(count=count.reshape(pH, pW, pw * ph), pack_start=start, data=data[:t],
                    index=index[:t])

    def pecr_conv(self, x, w, stride, pw, ph, ps, mode=0, workers=1):
        x, w = _f32(x), _f32(w)
        N, Cc, H, W = x.shape
        K, _, kh, kw = w.shape
        pH, pW = pack_dims(H, W, kh, kw, stride, pw, ph, ps)
        y = np.empty(N * K * pH * pW, np.float32)
        m, a = C.c_uint64(0), C.c_uint64(0)
        self._chk(self.lib.ref_pecr_conv(x.reshape(-1), N, Cc, H, W, w.reshape(-1), K, kh, kw,
                                         stride, pw, ph, ps, mode, workers, y, C.byref(m),
                                         C.byref(a)))
        return y.reshape(N, K, pH, pW), (m.value, a.value)

    def window_nnz(self, x, kh, kw, stride):
        x = _f32(x)
        Cc, H, W = x.shape
        oh, ow = out_dims(H, W, kh, kw, stride)
        out = np.empty(max(oh * ow, 1), np.int32)
        self._chk(self.lib.ref_window_nnz(x, Cc, H, W, kh, kw, stride, out))
        return out[:oh * ow].reshape(oh, ow)

    def checksum(self, v) -> str:
        v = _f32(v).reshape(-1)
        buf = C.create_string_buffer(17)
        self._chk(self.lib.ref_checksum(v, v.size, buf))
        return buf.value.decode()

    def plan(self, in_w, in_h, k_w, k_h, stride, channels, fmt=0, pw=0, ph=0, ps=1):
        b, t, s = C.c_int(), C.c_int(), C.c_uint64()
        self._chk(self.lib.ref_plan(in_w, in_h, k_w, k_h, stride, channels, fmt, pw, ph, ps,
                                    C.byref(b), C.byref(t), C.byref(s)))
        return b.value, t.value, s.value


def c_oracle() -> COracle:
    return COracle()


def ref_lib() -> RefLib | None:
    return RefLib() if os.path.exists(REF_SO) else None
