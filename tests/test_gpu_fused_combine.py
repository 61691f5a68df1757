"""Fused cross-GPU combine (b2_reduce_sum_fused) with two, four and eight processes. This
pool grants one GPU, so all ranks share cuda:0: the mailbox still crosses a process
boundary through a CUDA IPC mapping and the release/acquire protocol, the epoch
window and the bounded waits run exactly as across NVLink (the two contexts are
time-sliced, so this checks correctness, not speed). No barriers between the
iterations: ranks are free to race ahead up to the epoch window."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    from paper_2605_13864_b200 import shard
    fr = shard.FusedReduce()
    ok = True
    rng = np.random.default_rng(1000 + rank)
    results = []
    for it in range(12):
        n = 1_000_003 + 17 * it
        if it % 2 == 0:
            x = torch.from_numpy(rng.integers(-2**31, 2**31, n, dtype=np.int64).astype(np.int32)).cuda()
        else:
            x = torch.from_numpy(rng.uniform(-1, 1, n).astype(np.float32)).cuda()
        out = fr(x)
        torch.cuda.synchronize()
        local = x.to(torch.float64).sum().item() if x.dtype == torch.float32 else int(x.to(torch.int64).sum())
        results.append((it, float(out.item()) if x.dtype == torch.float32 else int(out.item()), local))
    # collect every rank's local sums on rank 0 and check the combined values
    allres = [None] * world
    dist.all_gather_object(allres, results)
    if rank == 0:
        for it in range(12):
            got = allres[0][it][1]
            want = sum(r[it][2] for r in allres)
            if it % 2 == 0:
                ok &= got == want
            else:
                ok &= abs(got - want) <= 1e-4 * max(1.0, abs(want))
        ok &= fr.status() == 0
    dist.barrier()
    fr.close()
    q.put((rank, bool(ok)))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4, 8])
def test_fused_combine_processes(world):
    """2, 4 and 8 ranks (the 8-GPU step's mailbox has one slot per rank and a window of
    epochs; more writers exercise the slot rows and the root's rank-order sum)."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    for p in ps:
        p.join(300)
        assert p.exitcode == 0
    res = dict(q.get() for _ in range(world))
    assert all(res[r] for r in range(world))


def test_timeout_does_not_poison_later_epochs():
    """a timed-out epoch used to leave the status word at 1 for
    ever. Now the status records the failed epoch, the root still releases the
    slot row, and the next healthy epoch reports 0 with the right sum."""
    import torch
    from paper_2605_13864_b200 import _lib, shard
    old = _lib.tuning("reduce.spin_ms")
    _lib.tune("reduce.spin_ms", 200)
    try:
        fr = shard.FusedReduce()  # no process group: rank 0 of 1
        x = torch.arange(1, 1001, dtype=torch.int32, device="cuda")
        fr.world = 2  # wait for a rank 1 that never publishes
        fr(x)
        torch.cuda.synchronize()
        assert fr.status() == 1 and fr.failed_epoch() == 1
        fr.world = 1
        for _ in range(6):  # past the 4-epoch slot window
            out = fr(x)
            torch.cuda.synchronize()
            assert int(out.item()) == 500500
            assert fr.status() == 0
        assert fr.failed_epoch() == 1
        fr.close()
    finally:
        _lib.tune("reduce.spin_ms", old)
