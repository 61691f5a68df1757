"""Multi-GPU partitioning of the two programs (one process per GPU,
torch.distributed for the plumbing).

The reference runs everything in one Python thread (interp.py:282-300 executes
`thread for` / `parallel for` sequentially); nothing in it is distributed. On
one 8 x B200 box the two programs shard as follows:

* transpose - row blocks, no exchange. Rank g owns input rows
  [r_g, r_{g+1}) (a multiple of the 64-row tile, the last block takes the
  remainder) and writes the W x (r_{g+1} - r_g) slab that is exactly
  out[:, r_g:r_{g+1}]. The output stays sharded; `gather_transpose` assembles
  it on one rank when a caller needs the whole matrix.
* reduction - contiguous shards plus one combine: each rank reduces its shard
  to one partial (int64 / float32) with the single-pass kernel, then
    int32 -> one NCCL reduce (sum) of the int64 partial to the root: exact in
             any order;
    fp32  -> one NCCL all-gather of the G partials, summed in rank order on
             every rank, so the result does not depend on NCCL's algorithm.
"""
from __future__ import annotations

import numpy as np

try:
    import torch
    import torch.distributed as dist
except Exception:  # pragma: no cover
    torch = dist = None


def row_blocks(H: int, world: int, align: int = 64) -> list:
    """[(r0, r1)] per rank: tile-aligned near-equal row blocks covering [0, H)."""
    if world <= 0:
        raise ValueError("world must be positive")
    units = -(-H // align) if H > 0 else 0
    base, extra = divmod(units, world)
    out, r = [], 0
    for g in range(world):
        nu = base + (1 if g < extra else 0)
        r1 = min(H, r + nu * align)
        out.append((r, r1))
        r = r1
    return out


def shard_range(n: int, world: int, rank: int, align: int = 4) -> tuple:
    """Contiguous [e0, e1) of an n-element array for `rank` (16-B aligned starts for
    4-byte cells when align = 4)."""
    blocks = row_blocks(n, world, align)
    return blocks[rank]


def _default_reduce(x):
    from . import ops
    return ops.reduce_sum(x)


def _default_transpose(a):
    from . import ops
    return ops.transpose(a)


def sharded_transpose(local_in, *, transpose_fn=None):
    """Transpose this rank's row block; returns the local W x H_g output slab."""
    return (transpose_fn or _default_transpose)(local_in)


def sharded_reduce_sum(local_x, *, group=None, root: int | None = None, reduce_fn=None):
    """Sum over all ranks' shards. int32 -> Python int (exact), float32 -> float
    (rank-order combine). With root=None every rank gets the result."""
    fn = reduce_fn or _default_reduce
    part = fn(local_x)
    is_int = str(getattr(local_x, "dtype", "")).endswith("int32")
    device = local_x.device if (torch is not None and isinstance(local_x, torch.Tensor)) else "cpu"
    if isinstance(part, (int, float, np.generic)):
        part = torch.tensor([part], dtype=torch.int64 if is_int else torch.float32, device=device)
    part = part.reshape(1)
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return int(part.item()) if is_int else float(part.item())
    if is_int:
        t = part.to(torch.int64)
        if root is None:
            dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
        else:
            dist.reduce(t, dst=root, op=dist.ReduceOp.SUM, group=group)
        return int(t.item())
    ws = dist.get_world_size(group)
    parts = [torch.empty_like(part) for _ in range(ws)]
    dist.all_gather(parts, part, group=group)
    acc = np.float32(0.0)
    for p in parts:  # rank order: deterministic
        acc = np.float32(acc + np.float32(p.item()))
    return float(acc)


class FusedReduce:
    """Sharded sum with the cross-GPU combine fused into the reduction kernel
    (include/b2k.h b2_reduce_sum_fused): no separate NCCL launch per step.

    Rank 0 owns a small mailbox in its HBM; its CUDA IPC handle is broadcast once
    over the process group (any backend) and opened by every other rank (a peer
    mapping over NVLink). Each call advances a shared epoch. The result on rank 0
    is the global sum (rank-ordered, deterministic for fp32); other ranks get
    their local partial.
    """

    def __init__(self, group=None, device=None):
        import ctypes

        from ._lib import check, lib
        self._lib, self._check, self._ct = lib(), check, ctypes
        self.group = group
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.dev = torch.cuda.current_device() if device is None else int(device)
        self.mailbox = ctypes.c_void_p()
        handle = ctypes.create_string_buffer(64)
        if self.rank == 0:
            check(self._lib.b2_mailbox_create(self.dev, ctypes.byref(self.mailbox), handle))
        obj = [handle.raw if self.rank == 0 else None]
        if self.world > 1:
            dist.broadcast_object_list(obj, src=0, group=group)
        if self.rank != 0:
            check(self._lib.b2_mailbox_open(obj[0], self.dev, ctypes.byref(self.mailbox)))
        self.epoch = 0

    def __call__(self, x, out=None, stream=None):
        from . import ops
        d = ops.b2_dtype(x)
        npacc, tacc = ops._ACC[d]
        if out is None:
            out = torch.empty(1, dtype=getattr(torch, tacc), device=x.device)
        self.epoch += 1
        self._check(self._lib.b2_reduce_sum_fused(
            x.data_ptr(), x.numel(), d, out.data_ptr(), None, 0, self.mailbox, self.rank, self.world,
            self.epoch, self.dev, ops._stream_ptr(x, stream)))
        return out

    def failed_epoch(self) -> int:
        """Latest epoch whose combine timed out on this rank's view (0 = never)."""
        s = self._ct.c_uint64(0)
        self._check(self._lib.b2_mailbox_status(self.mailbox, self.dev, self._ct.byref(s)))
        return int(s.value)

    def status(self) -> int:
        """Status of the latest call: 0 = healthy; 1 = a bounded wait of this epoch
        timed out (a rank never published). Earlier timeouts do not stick."""
        return 1 if self.epoch and self.failed_epoch() >= self.epoch else 0

    def close(self):
        if self.mailbox:
            self._lib.b2_mailbox_close(self.mailbox, self.dev, 1 if self.rank == 0 else 0)
            self.mailbox = self._ct.c_void_p()


def gather_transpose(local_out, rows: list, *, root: int = 0, group=None):
    """Assemble the full W x H output on `root` from the ranks' W x H_g slabs."""
    rank = dist.get_rank(group)
    ws = dist.get_world_size(group)
    W = local_out.shape[0]
    H = rows[-1][1]
    widths = [r1 - r0 for r0, r1 in rows]
    maxw = max(widths)
    buf = torch.zeros((W, maxw), dtype=local_out.dtype, device=local_out.device)
    buf[:, : local_out.shape[1]] = local_out
    bufs = [torch.empty_like(buf) for _ in range(ws)] if rank == root else None
    dist.gather(buf, bufs, dst=root, group=group)
    if rank != root:
        return None
    full = torch.empty((W, H), dtype=local_out.dtype, device=local_out.device)
    for (r0, r1), b in zip(rows, bufs):
        full[:, r0:r1] = b[:, : r1 - r0]
    return full
