"""Multi-rank host logic on CPU (gloo, world_size 2): batch shards cover the
batch exactly, the per-rank forward needs no collective, max-over-ranks timing
and the verification gather reconstruct the single-process result.  The
per-rank "forward" here is the CPU oracle (test infrastructure); on the B200
box bench.py runs the CUDA path with the same sharding code."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2002_00552_b200.sharding import gather_batch, max_over_ranks, shard_range


@pytest.mark.parametrize("n,world", [(1, 1), (7, 2), (8, 2), (512, 8), (3, 4), (1024, 8)])
def test_shard_range_partitions_batch(n, world):
    covered = []
    for r in range(world):
        a, b = shard_range(n, r, world)
        assert 0 <= a <= b <= n
        covered.extend(range(a, b))
    assert covered == list(range(n))
    sizes = [shard_range(n, r, world)[1] - shard_range(n, r, world)[0] for r in range(world)]
    assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_range(n, world, world)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle.dwm_oracle import draw, dwm_conv2d_oracle
        from paper_2002_00552_b200 import ConvSpec
        spec = ConvSpec(kernel=(5, 5), stride=(2, 2), pad=(2, 2, 2, 2))
        d, g = draw(3, (5, 5), (2, 2), 12, 3, 4, 5)
        a, b = shard_range(d.shape[0], rank, world)
        local = torch.from_numpy(dwm_conv2d_oracle(d[a:b], g, spec))     # no collective here
        full = gather_batch(local, d.shape[0], dist)
        slowest = max_over_ranks(0.5 + rank, dist)
        if rank == 0:
            ref = dwm_conv2d_oracle(d, g, spec)
            q.put((bool(np.array_equal(full.numpy(), ref)), slowest))
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_shard_gather_and_timing():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
    assert all(p.exitcode == 0 for p in procs)
    equal, slowest = q.get(timeout=5)
    assert equal
    assert slowest == 1.5
