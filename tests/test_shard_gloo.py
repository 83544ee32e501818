"""Multi-process (gloo, world_size 2 and 4) check of the 2-D C-tile sharding
used by bench.py --gpus N: panels broadcast from their owner ranks along
row / column groups, each rank multiplies its block (the C restatement stands
in for the GPU), and the gathered blocks equal the monolithic product
bit-for-bit (per-row / per-column scales make blocking exact)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2506_11277_b200 import shard


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, m, n, k, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import pyoracle as po
    blk = shard.block_of(rank, world, m, n)
    xchg = shard.PanelExchange(world, rank)  # the same exchange bench.py runs over NCCL
    # panels exist only on their owners (deterministic per-panel seeds)
    a = torch.zeros(blk.row1 - blk.row0, k, dtype=torch.float64)
    b = torch.zeros(k, blk.col1 - blk.col0, dtype=torch.float64)
    if rank == shard.a_owner(world, blk.i):
        a.copy_(torch.from_numpy(po.port_random_uniform(m, k, 1, -0.5, 0.5)[blk.row0:blk.row1]))
    if rank == shard.b_owner(world, blk.j):
        b.copy_(torch.from_numpy(po.port_random_uniform(k, n, 2, -0.5, 0.5)[:, blk.col0:blk.col1]))
    xchg.exchange(a, b)
    c = po.port_multiply_exact(a.numpy(), b.numpy(), 5, 4)
    out_q.put((rank, blk.row0, blk.row1, blk.col0, blk.col1, c))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4, 8])
def test_sharded_blocks_equal_monolithic(po, world):
    m, n, k = 40, 36, 50
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, m, n, k, q)) for r in range(world)]
    for p in procs:
        p.start()
    parts = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    c = np.full((m, n), np.nan)
    for _, r0, r1, c0, c1, blk in parts:
        c[r0:r1, c0:c1] = blk
    a = po.port_random_uniform(m, k, 1, -0.5, 0.5)
    b = po.port_random_uniform(k, n, 2, -0.5, 0.5)
    want = po.port_multiply_exact(a, b, 5, 4)
    assert np.array_equal(c.view(np.uint64), want.view(np.uint64))


def test_grid_and_groups():
    assert [shard.grid_for(w) for w in (1, 2, 4, 8)] == [(1, 1), (2, 1), (2, 2), (4, 2)]
    for w in (1, 2, 4, 8):
        blocks = [shard.block_of(r, w, 100, 70) for r in range(w)]
        cover = np.zeros((100, 70), dtype=int)
        for bl in blocks:
            cover[bl.row0:bl.row1, bl.col0:bl.col1] += 1
        assert (cover == 1).all()
        for bl in blocks:
            assert bl.rank in shard.row_group(w, bl.i) and bl.rank in shard.col_group(w, bl.j)
            assert shard.a_owner(w, bl.i) == shard.row_group(w, bl.i)[0]
