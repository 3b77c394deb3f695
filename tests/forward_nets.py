"""Seeded networks for the forward() parity tests.

Every filter bank and input comes from the reference generator
(sconv::generate, dataset.cpp:77-100) so the golden file only stores seeds,
checksums and counters.  `gen` is any object with generate(h, w, c, s, seed)
(the C oracle or the reference library: bit-identical).
"""
import numpy as np

# name -> (C, H, W, input sparsity, [(K, k, stride, relu, pool)]), pool = (pw, ph, ps, mode)
NETS = {
    # every branch of forward(): plain conv, fused conv+ReLU+max-pool, a pooled
    # layer without ReLU (PECR fallback, mean pool), a strided 2x2 conv
    "mixed": (3, 20, 20, 0.6, [(8, 3, 1, True, None), (6, 3, 1, True, (2, 2, 2, 0)),
                               (5, 3, 1, False, (2, 2, 2, 1)), (4, 2, 2, True, None)]),
    # VGG-style blocks (3x3 s1, K >= 32: the tiled kernels), ReLU sparsity
    "vgg_mini": (3, 36, 36, 0.0, [(32, 3, 1, True, None), (32, 3, 1, True, (2, 2, 2, 0)),
                                  (64, 3, 1, True, None), (64, 3, 1, True, (2, 2, 2, 0)),
                                  (128, 3, 1, True, None), (128, 3, 1, True, (2, 2, 2, 0))]),
    # LeNet-5 conv stack (5x5 kernels, 2x2 pools)
    "lenet": (1, 28, 28, 0.0, [(20, 5, 1, True, (2, 2, 2, 0)), (50, 5, 1, True, (2, 2, 2, 0))]),
    # overlapping 3x3/2 max pool after a 3x3 conv (AlexNet-style), then a 1x1 conv
    "overlap": (4, 17, 17, 0.5, [(16, 3, 1, True, (3, 3, 2, 0)), (8, 1, 1, True, None)]),
}
# PECR raises ConfigError on layer 0: Eq. 3 is not integral for 15 -> 13 with 2x2/2
BAD_PECR = (2, 15, 15, 0.5, [(8, 3, 1, True, (2, 2, 2, 0))])


def build(gen, spec, seed: int):
    """-> (x [C,H,W], layers) for image `seed` of a NETS entry."""
    C, H, W, s, layers = spec
    x = gen.generate(H, W, C, s, 1000 + seed)
    out, c = [], C
    for l, (K, k, stride, relu, pool) in enumerate(layers):
        f = np.stack([gen.generate(k, k, c, 0.0, 50_000 * (l + 1) + j) for j in range(K)])
        out.append({"filters": (f - np.float32(0.5)).astype(np.float32), "stride": stride,
                    "relu": relu, "pool": pool})
        c = K
    return x, out
