# Dev: would a tcgen05 3xTF32 (split hi/lo) dense conv meet the FAST parity bar?
# Emulates one MMA k-step (8 products, exact, one rounding into the fp32
# accumulator) against the reference order (sequential fp32 mul then add over
# (c, i, j), src/ecr.cpp:117-120), and prints max |err| / (1e-5 + 1e-5|ref|).
# Usage: python tools/tf32_feasibility.py C   (C = input channels)
import numpy as np, sys
rng = np.random.default_rng(1)
C, K, H = int(sys.argv[1]), 16, 20
x = rng.random((C, H + 2, H + 2), dtype=np.float32)
x *= (rng.random(x.shape) >= 0.7)
w = (rng.random((K, C, 3, 3), dtype=np.float32) - 0.5).astype(np.float32)
def tf32(a):  # round-to-nearest to 10 mantissa bits
    u = a.astype(np.float32).view(np.uint32).astype(np.uint64)
    u = ((u + 0x1000) & ~np.uint64(0x1FFF)).astype(np.uint32)
    return u.view(np.float32)
# im2col: [H*H, C*9] in (c,i,j) order
cols = np.stack([x[c, i:i + H, j:j + H].reshape(-1) for c in range(C) for i in range(3) for j in range(3)], 1)
Wm = w.reshape(K, -1).T  # [C*9, K]
# reference: sequential fp32, mul then add, (c,i,j) order
ref = np.zeros((H * H, K), np.float32)
for p in range(cols.shape[1]):
    ref = (ref + (cols[:, p:p + 1] * Wm[p:p + 1, :]).astype(np.float32)).astype(np.float32)
def emu(passes, kchunk=8):
    ah, bh = tf32(cols), tf32(Wm)
    al, bl = tf32(cols - ah), tf32(Wm - bh)
    terms = {1: [(ah, bh)], 3: [(al, bh), (ah, bl), (ah, bh)]}[passes]
    acc = np.zeros((H * H, K), np.float32)
    for a, b in terms:
        for k0 in range(0, a.shape[1], kchunk):  # one MMA k-step: exact products, fp64 sum, one rounding
            part = a[:, k0:k0 + kchunk].astype(np.float64) @ b[k0:k0 + kchunk].astype(np.float64)
            acc = (acc.astype(np.float64) + part).astype(np.float32)
    return acc
bar = 1e-5 + 1e-5 * np.abs(ref)
for ps in (1, 3):
    print("C", C, "passes", ps, "max err / bar", float((np.abs(emu(ps) - ref) / bar).max()))
# FFMA order (our FAST): fma in (c,i,j) order
acc = np.zeros((H * H, K), np.float32)
for p in range(cols.shape[1]):
    acc = (acc.astype(np.float64) + cols[:, p:p+1].astype(np.float64) * Wm[p:p+1].astype(np.float64)).astype(np.float32)
print("C", C, "FFMA (c,i,j) max err / bar", float((np.abs(acc - ref) / bar).max()))
