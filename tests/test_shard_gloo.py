"""N > 1 path on CPU: world_size-2 gloo process groups exercise the row-block
and shard partitioning and the partial combine. The per-rank compute is
injected from the CPU oracle (these tests check the partition/combine logic;
the per-rank kernels are covered by the -m gpu tests)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle
from paper_2605_13864_b200 import shard


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, kind, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(42)
        if kind == "transpose":
            H, W = 300, 77
            a = rng.standard_normal((H, W)).astype(np.float32)
            rows = shard.row_blocks(H, world)
            r0, r1 = rows[rank]
            local = shard.sharded_transpose(a[r0:r1], transpose_fn=lambda x: torch.from_numpy(oracle.transpose(x)))
            full = shard.gather_transpose(local, rows, root=0)
            if rank == 0:
                q.put(("transpose", bool(np.array_equal(full.numpy(), a.T))))
        elif kind == "reduce_int":
            n = 100_003
            x = rng.integers(-2**31, 2**31, n, dtype=np.int64).astype(np.int32)
            e0, e1 = shard.shard_range(n, world, rank)
            tot = shard.sharded_reduce_sum(torch.from_numpy(x[e0:e1]),
                                           reduce_fn=lambda t: oracle.reduce_i32(t.numpy()))
            q.put(("reduce_int", rank, tot == int(x.astype(np.int64).sum())))
        else:
            n = 65_537
            x = rng.uniform(-1, 1, n).astype(np.float32)
            e0, e1 = shard.shard_range(n, world, rank)
            tot = shard.sharded_reduce_sum(torch.from_numpy(x[e0:e1]),
                                           reduce_fn=lambda t: oracle.reduce_f32_seq(t.numpy()))
            # deterministic rank-order combine of the per-rank partials
            parts = [oracle.reduce_f32_seq(x[a:b]) for a, b in shard.row_blocks(n, world, 4)]
            want = np.float32(0)
            for p in parts:
                want = np.float32(want + np.float32(p))
            exact, absum = oracle.sum_f64(x)
            q.put(("reduce_f32", rank, tot == float(want) and
                   abs(tot - exact) <= oracle.f32_tolerance(n, exact, absum)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("kind", ["transpose", "reduce_int", "reduce_f32"])
def test_world2_gloo(kind):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, kind, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    res = []
    while not q.empty():
        res.append(q.get())
    assert res and all(r[-1] for r in res), res


@pytest.mark.parametrize("H,world", [(0, 2), (1, 2), (64, 8), (32768, 8), (1000, 3), (65, 2)])
def test_row_blocks_cover_exactly(H, world):
    rows = shard.row_blocks(H, world)
    assert len(rows) == world
    assert rows[0][0] == 0 and rows[-1][1] == H
    for (a, b), (c, d) in zip(rows, rows[1:]):
        assert b == c and a <= b
    assert all(r0 % 64 == 0 for r0, r1 in rows if r1 > r0)
