"""Multi-GPU partition for the ECR / PECR path (one process per GPU).

Images are independent and output channels are independent given the full
input, so the (image, filter) grid is split with no collective on the data
path: rank r of W owns the contiguous shard returned by sconv_shard -- images
when N >= W, otherwise output channels (include/sconv_cuda.h).  This is the
multi-GPU analogue of dispatch's contiguous block-row partition
(include/sconv/exec.hpp:89-107).  Each output is produced by exactly one rank
with the same per-output arithmetic, so results are bit-identical for every
world size.
"""
from __future__ import annotations

import os
from dataclasses import dataclass

from .api import shard


@dataclass(frozen=True)
class Shard:
    rank: int
    world: int
    n_begin: int
    n_end: int
    k_begin: int
    k_end: int

    @property
    def images(self) -> int:
        return self.n_end - self.n_begin

    @property
    def filters(self) -> int:
        return self.k_end - self.k_begin


def shard_for(n: int, k: int, world: int, rank: int) -> Shard:
    return Shard(rank, world, *shard(n, k, world, rank))


def env_rank_world() -> tuple[int, int, int]:
    """(rank, world, local_rank) from the torchrun environment."""
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def assemble(parts, n: int, k: int, world: int):
    """Reassemble per-rank outputs [n_r, k_r, ...] (rank order) into [n, k, ...]
    (numpy or torch); used by gather-side callers and tests."""
    import numpy as np
    first = parts[0]
    is_np = isinstance(first, np.ndarray)
    tail = tuple(first.shape[2:])
    if is_np:
        out = np.empty((n, k) + tail, first.dtype)
    else:
        import torch
        out = torch.empty((n, k) + tail, dtype=first.dtype, device=first.device)
    for r, p in enumerate(parts):
        s = shard_for(n, k, world, r)
        if s.images and s.filters:
            out[s.n_begin:s.n_end, s.k_begin:s.k_end] = p
    return out
