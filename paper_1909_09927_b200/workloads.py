"""The benchmark workloads of BASELINE.json, shared by bench.py and the tests.

VGG-19's 16 conv layers as SURVEY.md 8(d) defines them: valid 3x3 stride-1
convolution on pre-padded (H+2)x(W+2) inputs (so the outputs are VGG's HxW),
the 5 layers followed by a 2x2/2 max pool marked `pooled` (forward's fused
PECR branch, src/pipeline.cpp:249-264).  Inputs come from the reference's
generator (src/dataset.cpp:77-100, bit-identical sconv_generate):

    map  n of layer l:  generate(H+2, W+2, C, s, 1e6*(l+1) + n)
    filt k of layer l:  generate(3, 3, C, 0, 1e6*(l+1) + 5e5 + k) - 0.5
"""
from __future__ import annotations

from typing import Optional, Sequence

import numpy as np

# (name, C, K, H_out, pooled?)
VGG19 = [
    ("conv1_1", 3, 64, 224, False), ("conv1_2", 64, 64, 224, True),
    ("conv2_1", 64, 128, 112, False), ("conv2_2", 128, 128, 112, True),
    ("conv3_1", 128, 256, 56, False), ("conv3_2", 256, 256, 56, False),
    ("conv3_3", 256, 256, 56, False), ("conv3_4", 256, 256, 56, True),
    ("conv4_1", 256, 512, 28, False), ("conv4_2", 512, 512, 28, False),
    ("conv4_3", 512, 512, 28, False), ("conv4_4", 512, 512, 28, True),
    ("conv5_1", 512, 512, 14, False), ("conv5_2", 512, 512, 14, False),
    ("conv5_3", 512, 512, 14, False), ("conv5_4", 512, 512, 14, True),
]
SWEEP = (0.5, 0.6, 0.7, 0.8, 0.9, 0.95)


def map_seed(l: int, n: int) -> int:
    return 1_000_000 * (l + 1) + n


def filt_seed(l: int, k: int) -> int:
    return 1_000_000 * (l + 1) + 500_000 + k


def vgg_maps(l: int, images: Sequence[int], sparsity: float,
             out: Optional[np.ndarray] = None) -> np.ndarray:
    """Input maps [len(images), C, H+2, H+2] of layer l for the given image ids."""
    from .api import generate_batch
    _, C, _, H, _ = VGG19[l]
    return generate_batch([map_seed(l, n) for n in images], H + 2, H + 2, C, sparsity, out=out)


def vgg_filters(l: int, ks: Optional[Sequence[int]] = None,
                out: Optional[np.ndarray] = None) -> np.ndarray:
    """Filters [len(ks), C, 3, 3] of layer l (all K when ks is None), minus 0.5."""
    from .api import generate_batch
    _, C, K, _, _ = VGG19[l]
    ks = range(K) if ks is None else ks
    w = generate_batch([filt_seed(l, k) for k in ks], 3, 3, C, 0.0, out=out)
    w -= np.float32(0.5)
    return w
