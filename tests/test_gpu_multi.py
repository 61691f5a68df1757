"""Single-process multi-GPU entries (b2_transpose_multi / b2_reduce_sum_multi,
SURVEY 8b/8e). Shards go to every visible GPU round-robin; on a one-GPU box
several shards share cuda:0, which runs the same code (same-device combine
through the root's mailbox, launch ordering that keeps the root's wait from
blocking its co-resident shards)."""
import numpy as np
import pytest
import torch

import paper_2605_13864_b200 as b2
from oracle import oracle

pytestmark = pytest.mark.gpu


def _devs(k):
    n = torch.cuda.device_count()
    return [torch.device("cuda", g % n) for g in range(k)]


def _row_blocks(rows, k, tile=64):
    """SURVEY 8e split: whole tiles per shard, the last one takes the remainder."""
    per = -(-rows // k)
    per = -(-per // tile) * tile
    cuts = [min(rows, g * per) for g in range(k + 1)]
    cuts[-1] = rows
    return cuts


@pytest.mark.parametrize("shape,dt,k", [((1000, 777), np.float32, 3), ((4096, 2048), np.float32, 4),
                                        ((640, 384), np.uint16, 2), ((300, 130), np.float64, 5),
                                        ((129, 65), np.float32, 8)])
def test_transpose_multi_sharded_outputs(shape, dt, k):
    rng = np.random.default_rng(11)
    a = rng.integers(0, 2**16, shape).astype(dt)
    cuts = _row_blocks(shape[0], k)
    devs = _devs(k)
    shards = [torch.from_numpy(a[cuts[g]:cuts[g + 1]].copy()).to(devs[g]) for g in range(k)]
    outs = b2.transpose_multi(shards)
    want = oracle.transpose(a)
    for g in range(k):
        assert np.array_equal(outs[g].cpu().numpy(), want[:, cuts[g]:cuts[g + 1]]), g


def test_transpose_multi_into_one_full_matrix():
    """Column-slab views of one full output on the root: the shards' kernels
    write their slabs in place (over NVLink when the shard is on another GPU)."""
    rng = np.random.default_rng(12)
    a = rng.standard_normal((2048, 1536)).astype(np.float32)
    k = 4
    cuts = _row_blocks(2048, k)
    devs = _devs(k)
    shards = [torch.from_numpy(a[cuts[g]:cuts[g + 1]].copy()).to(devs[g]) for g in range(k)]
    full = torch.empty((1536, 2048), dtype=torch.float32, device="cuda:0")
    b2.transpose_multi(shards, [full[:, cuts[g]:cuts[g + 1]] for g in range(k)])
    assert np.array_equal(full.cpu().numpy(), oracle.transpose(a))


@pytest.mark.parametrize("k", [1, 2, 3, 8])
def test_reduce_multi_int32_exact(k):
    rng = np.random.default_rng(20 + k)
    x = rng.integers(-2**31, 2**31, 3_000_001, dtype=np.int64).astype(np.int32)
    cuts = np.linspace(0, x.size, k + 1).astype(np.int64)
    devs = _devs(k)
    shards = [torch.from_numpy(x[cuts[g]:cuts[g + 1]].copy()).to(devs[g]) for g in range(k)]
    for _ in range(6):  # > the mailbox's 4-epoch window
        assert b2.reduce_sum_multi(shards) == oracle.reduce_i32(x)


def test_reduce_multi_with_empty_and_ragged_shards():
    rng = np.random.default_rng(30)
    sizes = [0, 1, 5, 1 << 20, 0, 777]
    devs = _devs(len(sizes))
    xs = [rng.integers(-2**31, 2**31, s, dtype=np.int64).astype(np.int32) for s in sizes]
    shards = [torch.from_numpy(v).to(d) for v, d in zip(xs, devs)]
    assert b2.reduce_sum_multi(shards) == sum(int(v.astype(np.int64).sum()) for v in xs)


@pytest.mark.parametrize("dt", [np.float32, np.float64])
def test_reduce_multi_float_rank_order(dt):
    """fp32 / fp64: the combine sums the per-shard partials in shard order, so the
    result is bit-identical to summing the single-GPU results in that order, and
    within the north-star tolerance of the exact sum."""
    rng = np.random.default_rng(40)
    x = rng.uniform(-1, 1, 5_000_003).astype(dt)
    k = 4
    cuts = np.linspace(0, x.size, k + 1).astype(np.int64)
    devs = _devs(k)
    shards = [torch.from_numpy(x[cuts[g]:cuts[g + 1]].copy()).to(devs[g]) for g in range(k)]
    got = b2.reduce_sum_multi(shards)
    parts = [b2.reduce_sum(s).item() for s in shards]
    acc = dt(0)
    for p in parts:
        acc = dt(acc + dt(p))
    assert dt(got) == acc
    exact, absum = oracle.sum_f64(x.astype(np.float32)) if dt == np.float32 else (float(np.sum(x)), float(np.abs(x).sum()))
    if dt == np.float32:
        assert abs(got - exact) <= oracle.f32_tolerance(x.size, exact, absum)
    else:
        assert abs(got - exact) <= 1e-9 * absum


def test_peer_access_and_init():
    b2.init_devices()
    from paper_2605_13864_b200 import _lib
    assert _lib.lib().b2_peer_access(0, 0) == 1
