"""World-size-2 gloo run of the multi-GPU partition on CPU.

Each rank takes its sconv_shard of the (image, filter) grid, computes it with
the checker (the C oracle stands in for the per-rank device work, there is
no GPU here), and the shards are all-gathered and reassembled: the result
must equal the single-process output bit for bit, for both the image split
(N >= world) and the output-channel split (N < world).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, k, kind, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle.oracle import c_oracle
        from paper_1909_09927_b200.partition import assemble, shard_for
        orc = c_oracle()
        x = np.stack([orc.generate(14, 14, 5, 0.7, 50 + i) for i in range(n)])
        w = np.stack([orc.generate(3, 3, 5, 0.0, 90 + j) for j in range(k)]) - np.float32(0.5)
        s = shard_for(n, k, world, rank)
        xs, ws = x[s.n_begin:s.n_end], w[s.k_begin:s.k_end]
        if kind == "ecr":
            part, ops = orc.ecr_conv(xs, ws, 1)
        else:
            part, ops = orc.pecr_conv(xs, ws, 1, 2, 2, 2, 0)
        parts = [None] * world
        dist.all_gather_object(parts, part)
        tot = torch.tensor([ops[0], ops[1]], dtype=torch.int64)
        dist.all_reduce(tot)
        if rank == 0:
            full = assemble(parts, n, k, world)
            ref, rops = orc.ecr_conv(x, w, 1) if kind == "ecr" else orc.pecr_conv(x, w, 1, 2, 2, 2, 0)
            q.put((np.array_equal(full.view(np.uint32), ref.view(np.uint32)),
                   tuple(tot.tolist()) == rops))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n,k,kind", [(4, 6, "ecr"), (1, 6, "ecr"), (3, 4, "pecr"), (1, 5, "pecr")])
def test_gloo_world2(n, k, kind):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n, k, kind, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    same, ops_ok = q.get(timeout=5)
    assert same and ops_ok


def _gpu_worker(rank, world, port, n, k, kind, q):
    """Same partition, but each rank computes its shard on the GPU (both
    ranks share cuda:0 here: one process per GPU on a node, one GPU in CI)."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1909_09927_b200 as sc
        from oracle.oracle import c_oracle
        from paper_1909_09927_b200.partition import assemble, shard_for
        orc = c_oracle()
        x = np.stack([orc.generate(22, 22, 16, 0.7, 60 + i) for i in range(n)])
        w = np.stack([orc.generate(3, 3, 16, 0.0, 95 + j) for j in range(k)]) - np.float32(0.5)
        s = shard_for(n, k, world, rank)
        xs, ws = x[s.n_begin:s.n_end], w[s.k_begin:s.k_end]
        ops = sc.OpCount()
        if kind == "ecr":
            part = sc.ecr_conv_batched(xs, ws, 1, counters=ops, device=0)
        else:
            part = sc.pecr_conv_pool_batched(xs, ws, 1, sc.PoolConfig(2, 2, 2), counters=ops,
                                             device=0)
        parts = [None] * world
        dist.all_gather_object(parts, part)
        tot = torch.tensor([ops.multiplications, ops.additions], dtype=torch.int64)
        dist.all_reduce(tot)
        if rank == 0:
            full = assemble(parts, n, k, world)
            ref, rops = orc.ecr_conv(x, w, 1) if kind == "ecr" else orc.pecr_conv(x, w, 1, 2, 2, 2, 0)
            q.put((np.array_equal(full.view(np.uint32), ref.view(np.uint32)),
                   tuple(tot.tolist()) == rops))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("n,k,kind", [(4, 128, "ecr"), (1, 128, "ecr"), (3, 64, "pecr")])
def test_gloo_world2_device(n, k, kind):
    """World size 2 with the per-rank compute on the GPU: the gathered result
    is bit-identical to the oracle and the counters sum to its OpCount."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gpu_worker, args=(r, 2, port, n, k, kind, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(300)
        assert p.exitcode == 0
    same, ops_ok = q.get(timeout=5)
    assert same and ops_ok
