"""Small, torch-free workload that exercises every libb200k kernel, for
compute-sanitizer (memcheck / racecheck / synccheck / initcheck).

The reference's static guarantees (checker.py: E-DESYNC for accesses into a
desynchronised group without a barrier, :447-452; E-THREADS-CTX for barriers not
executed block-wide, :782-789) have their runtime analogue here: racecheck and
synccheck over the hand-written kernels, memcheck/initcheck over their
addressing. Every case also checks its result bit-exact (transposes, integer
sums, A.5 tree order) or within the north-star tolerance (fp32 sums), so a
sanitizer run is also a parity run.

    python tools/sanitize_driver.py [transpose|transpose_big|reduce|fused|multi|codegen|all]

Used by tests/test_gpu_sanitizer.py; needs a GPU, no torch CUDA context.
"""
from __future__ import annotations

import ctypes
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2605_13864_b200 import _lib  # noqa: E402
from paper_2605_13864_b200._lib import check, lib  # noqa: E402

L = lib()
DEV = 0
DT = {np.dtype(np.float32): _lib.F32, np.dtype(np.float64): _lib.F64, np.dtype(np.uint16): _lib.BF16,
      np.dtype(np.int32): _lib.I32, np.dtype(np.uint8): _lib.U8}


def dalloc(nbytes: int) -> int:
    p = ctypes.c_void_p()
    check(L.b2_device_alloc(max(nbytes, 1), DEV, ctypes.byref(p)))
    return p.value


def dfree(p: int) -> None:
    check(L.b2_device_free(p, DEV))


def h2d(a: np.ndarray) -> int:
    p = dalloc(a.nbytes)
    check(L.b2_copy_h2d(p, a.ctypes.data, a.nbytes, DEV))
    return p


def d2h(p: int, like: np.ndarray) -> np.ndarray:
    out = np.empty_like(like)
    check(L.b2_copy_d2h(out.ctypes.data, p, out.nbytes, DEV))
    return out


def tune(key, val):
    check(L.b2_tune_set(key.encode(), val))


def rand(shape, dt, rng):
    if dt == np.float32:
        return rng.uniform(-1, 1, shape).astype(np.float32)
    if dt == np.float64:
        return rng.standard_normal(shape)
    return rng.integers(0, np.iinfo(dt).max, shape, dtype=np.int64).astype(dt)


def one_transpose(rows, cols, dt, rng, pad_in=0, pad_out=0, off=0):
    """Device-entry transpose of a (rows x cols) view with pitches cols+pad_in /
    rows+pad_out, base shifted by `off` elements; the padding is left untouched."""
    ld_in, ld_out = cols + pad_in, rows + pad_out
    full = rand((rows * ld_in + off,), dt, rng)
    a = full[off:].reshape(rows, ld_in)[:, :cols]
    guard = rand((cols * ld_out + off,), dt, rng)
    pin, pout = h2d(full), h2d(guard)
    es = full.itemsize
    check(L.b2_transpose(pin + off * es, pout + off * es, rows, cols, ld_in, ld_out,
                         DT[np.dtype(dt)], DEV, None))
    got = d2h(pout, guard)
    want = guard.copy()
    want[off:].reshape(cols, ld_out)[:, :rows] = a.T
    assert np.array_equal(got.view(np.uint8), want.view(np.uint8)), (rows, cols, dt, pad_in, pad_out, off)
    dfree(pin)
    dfree(pout)


def run_transpose(rng):
    # vector tiles: fp32 64x64, bf16 128x128 (prmt repack), fp64 64x32; edges + ragged
    for rows, cols, dt in [(256, 384, np.float32), (250, 390, np.float32), (256, 512, np.uint16),
                           (130, 66, np.float64), (1, 1, np.float32), (1, 3000, np.float32),
                           (3000, 1, np.float32), (5, 7, np.uint8), (33, 65, np.uint16)]:
        one_transpose(rows, cols, dt, rng)
    # odd pitches / misaligned bases -> cp.async-staged kernel (every ring depth), the
    # padded scalar tile, then the funnel-shift path
    tune("transpose.staged", 2)
    for stages in (4, 3, 2):
        tune("transpose.staged_stages", stages)
        one_transpose(200, 300, np.float32, rng, pad_in=1, pad_out=3)
        one_transpose(130, 390, np.uint16, rng, pad_in=1, pad_out=1)
        one_transpose(70, 45, np.float64, rng, pad_in=1, pad_out=3)
    tune("transpose.staged_stages", 4)
    for geom in range(1, 6):  # 128 / 256-row tiles, ring depths, the evict-first hint
        tune("transpose.staged_geom", geom)
        one_transpose(300, 130, np.float32, rng, pad_in=1, pad_out=3)
        one_transpose(270, 260, np.uint16, rng, pad_in=3, pad_out=1)
    tune("transpose.staged_geom", 0)
    one_transpose(128, 96, np.float32, rng, off=1)
    one_transpose(120, 88, np.uint16, rng, pad_in=3, off=1)
    tune("transpose.staged", 0)
    one_transpose(200, 300, np.float32, rng, pad_in=1, pad_out=3)
    one_transpose(120, 88, np.uint16, rng, pad_in=3, off=1)
    tune("transpose.staged", 1)
    tune("transpose.any", 1)
    one_transpose(200, 300, np.float32, rng, pad_in=1, pad_out=3)
    one_transpose(128, 96, np.float64, rng, pad_in=1)
    tune("transpose.any", 0)
    # every fp32 tile variant (incl. the 128-KB tile the bench uses on large matrices)
    for v in range(11):
        tune("transpose.variant", v)
        one_transpose(512, 640, np.float32, rng)
    tune("transpose.variant", 0)
    for v in (1, 2, 7):
        tune("transpose.variant", v)
        one_transpose(384, 320, np.uint16, rng)
        one_transpose(300, 200, np.float64, rng)
    tune("transpose.variant", 0)
    # the 128-KB fp32 / fp64 tiles (auto-selected on >= 8 x #SM tiles; forced here)
    tune("transpose.big", 2)
    one_transpose(520, 300, np.float32, rng)
    one_transpose(600, 130, np.float64, rng)
    tune("transpose.big", 1)
    # cp.async-loaded tiles (the default on large matrices; forced here, every geometry,
    # every cell width, ragged tiles, pitched / offset views)
    tune("transpose.cpa", 2)
    for v in range(10):
        tune("transpose.cpa_variant", v)
        one_transpose(520, 300, np.float32, rng, pad_in=4, pad_out=8)
        one_transpose(264, 136, np.uint16, rng, pad_in=8)
        one_transpose(200, 70, np.float64, rng, pad_out=2)
    tune("transpose.cpa_variant", 0)
    tune("transpose.cpa", 1)
    # TMA-staged variants: 1 = UTMALDG/UTMASTG + mbarrier ring; 2 = TMA-loaded
    # input stages, register transpose, direct stores (all stage counts)
    tune("transpose.tma", 1)
    one_transpose(1024, 768, np.float32, rng)
    one_transpose(1000, 770, np.float32, rng)
    tune("transpose.tma", 2)
    for stages in (2, 3, 4, 6):
        tune("transpose.tma_stages", stages)
        one_transpose(1024, 768, np.float32, rng)
        one_transpose(1000, 772, np.float32, rng)
    tune("transpose.tma_stages", 2)
    tune("transpose.tma", 0)
    # host pipeline (chunked H2D / kernel / D2H) with a small stage size
    tune("host.chunk_mb", 1)
    a = rand((1500, 1100), np.float32, rng)
    out = np.empty((1100, 1500), np.float32)
    check(L.b2_transpose_host(a.ctypes.data, out.ctypes.data, 1500, 1100, 1100, 1500, _lib.F32, DEV))
    assert np.array_equal(out, a.T)
    tune("host.chunk_mb", 0)


def run_reduce(rng):
    sys.path.insert(0, ROOT)
    from oracle import oracle
    for n in [1, 3, 4, 1000, 4099, (1 << 20) + 5]:
        xi = rng.integers(-2**31, 2**31, n + 1, dtype=np.int64).astype(np.int32)
        for off in (0, 1):
            x = xi[off:off + n]
            p = h2d(np.ascontiguousarray(x))
            res = np.zeros(1, np.int64)
            outp = dalloc(8)
            check(L.b2_reduce_sum(p, n, _lib.I32, outp, None, 0, DEV, None))
            got = d2h(outp, res)[0]
            assert int(got) == int(x.astype(np.int64).sum()), n
            dfree(p)
            dfree(outp)
        xf = rng.uniform(-1, 1, n).astype(np.float32)
        p = h2d(xf)
        wsb = int(L.b2_reduce_ws_bytes(n, _lib.F32))
        ws = dalloc(wsb)
        zeros = np.zeros(wsb, np.uint8)  # keep the host buffer alive across the call
        check(L.b2_copy_h2d(ws, zeros.ctypes.data, wsb, DEV))
        outp = dalloc(4)
        for _ in range(2):  # the kernel re-arms its own workspace
            check(L.b2_reduce_sum(p, n, _lib.F32, outp, ws, wsb, DEV, None))
            got = float(d2h(outp, np.zeros(1, np.float32))[0])
            exact, absum = oracle.sum_f64(xf)
            assert abs(got - exact) <= oracle.f32_tolerance(n, exact, absum), n
        dfree(p)
        dfree(ws)
        dfree(outp)
    # the naive fp32 program in the reference's order (one warp, 4-byte cp.async ring),
    # device entry on a misaligned view and the chunked host entry; bit-exact
    for n in [0, 1, 5, 2048, 2049, 10007]:
        xf = rng.uniform(-1, 1, n + 1).astype(np.float32)
        want = np.cumsum(xf[1:], dtype=np.float32)[-1] if n else np.float32(0)
        p = h2d(xf)
        acc = h2d(np.zeros(1, np.float32))
        check(L.b2_reduce_sum_seq_f32(p + 4, n, acc, DEV, None))
        assert d2h(acc, np.zeros(1, np.float32))[0].view(np.uint32) == want.view(np.uint32), n
        res = np.zeros(1, np.float32)
        check(L.b2_reduce_sum_seq_f32_host(xf[1:].ctypes.data, n, res.ctypes.data, DEV))
        assert res[0].view(np.uint32) == want.view(np.uint32), n
        dfree(p)
        dfree(acc)
    # every reduce variant
    x = rng.integers(-2**31, 2**31, 300_001, dtype=np.int64).astype(np.int32)
    p = h2d(x)
    outp = dalloc(8)
    for v in range(10):  # incl. the 256-bit-load variants (LDG.E.256)
        tune("reduce.variant", v)
        check(L.b2_reduce_sum(p, x.size, _lib.I32, outp, None, 0, DEV, None))
        assert int(d2h(outp, np.zeros(1, np.int64))[0]) == int(x.astype(np.int64).sum()), v
    tune("reduce.variant", 0)
    dfree(p)
    dfree(outp)
    # A.5 tree order: partials bit-exact, then the host pipeline
    xf = rng.uniform(-1, 1, 512 * 700).astype(np.float32)
    p = h2d(xf)
    parts = dalloc(700 * 4)
    check(L.b2_reduce_tree512_partials(p, xf.size, parts, DEV, None))
    got = d2h(parts, np.zeros(700, np.float32))
    want_total, want_parts = oracle.reduce_f32_tree512(xf)
    assert np.array_equal(got, np.asarray(want_parts, np.float32))
    res = ctypes.c_float()
    check(L.b2_reduce_tree512_host(xf.ctypes.data, xf.size, ctypes.byref(res), DEV))
    assert np.float32(res.value) == np.float32(want_total)
    dfree(p)
    dfree(parts)
    # the A.5 family: every tree block size
    for blk in (64, 128, 256, 1024, 2048):
        xb = rng.uniform(-1, 1, blk * 37).astype(np.float32)
        pb = h2d(xb)
        parts = dalloc(37 * 4)
        check(L.b2_reduce_tree_partials(pb, xb.size, blk, parts, DEV, None))
        d2h(parts, np.zeros(37, np.float32))
        dfree(pb)
        dfree(parts)
    # host pipeline, int32, small stage size
    tune("host.chunk_mb", 1)
    x = rng.integers(-2**31, 2**31, 3_000_017, dtype=np.int64).astype(np.int32)
    r = np.zeros(1, np.int64)
    check(L.b2_reduce_sum_host(x.ctypes.data, x.size, _lib.I32, r.ctypes.data, DEV))
    assert int(r[0]) == int(x.astype(np.int64).sum())
    tune("host.chunk_mb", 0)


def run_fused(rng):
    """Single-rank fused combine: the mailbox protocol end to end (rank 0 is both
    writer and root), several epochs."""
    mb = ctypes.c_void_p()
    handle = ctypes.create_string_buffer(64)
    check(L.b2_mailbox_create(DEV, ctypes.byref(mb), handle))
    for epoch in range(1, 7):
        x = rng.integers(-2**31, 2**31, 100_000 + epoch, dtype=np.int64).astype(np.int32)
        p = h2d(x)
        outp = dalloc(8)
        check(L.b2_reduce_sum_fused(p, x.size, _lib.I32, outp, None, 0, mb, 0, 1, epoch, DEV, None))
        assert int(d2h(outp, np.zeros(1, np.int64))[0]) == int(x.astype(np.int64).sum())
        dfree(p)
        dfree(outp)
    st = ctypes.c_uint64()
    check(L.b2_mailbox_status(mb, DEV, ctypes.byref(st)))
    assert st.value == 0
    check(L.b2_mailbox_close(mb, DEV, 1))


def run_codegen(rng):
    """Generated kernels (codegen.py) for the GPU-form programs A.4 / A.5."""
    import paper_2605_13864_b200 as b2
    tp = b2.parse_program(b2.programs.TRANSPOSE_GPU)
    m = rng.standard_normal((64, 96)).astype(np.float32)
    _, outs = b2.run_program(tp, "transpose", {"in": b2.Array([64, 96], m.reshape(-1).tolist(), "float"),
                                               "out": b2.Array.alloc([96, 64], "float"), "W": 96, "H": 64},
                             backend="codegen")
    assert outs["out"] == m.T.reshape(-1).tolist()
    rp = b2.parse_program(b2.programs.REDUCE_TREE)
    x = rng.uniform(-1, 1, 2048).astype(np.float32)
    from oracle import oracle
    ret, _ = b2.run_program(rp, "reduce", {"arr": x.tolist(), "N": 2048}, backend="codegen")
    assert np.float32(ret) == np.float32(oracle.reduce_f32_tree512(x)[0])


def run_transpose_big(rng):
    """The 128-KB tiles as auto-selected on a real-size matrix (memcheck only)."""
    one_transpose(256 * 37, 128 * 32 + 40, np.float32, rng)
    one_transpose(256 * 37, 64 * 32 + 24, np.float64, rng)


def run_multi(rng):
    """Single-process multi-shard entries (all shards on device 0 here)."""
    k = 3
    a = rand((300, 200), np.float32, rng)
    cuts = [0, 128, 256, 300]
    ins = [h2d(np.ascontiguousarray(a[cuts[g]:cuts[g + 1]])) for g in range(k)]
    outs = [dalloc(200 * (cuts[g + 1] - cuts[g]) * 4) for g in range(k)]
    rows = [cuts[g + 1] - cuts[g] for g in range(k)]
    vp = ctypes.c_void_p * k
    i64 = ctypes.c_int64 * k
    check(L.b2_transpose_multi(vp(*ins), vp(*outs), i64(*rows), 200, i64(*[200] * k), i64(*rows), _lib.F32, k))
    for g in range(k):
        got = d2h(outs[g], np.empty((200, rows[g]), np.float32))
        assert np.array_equal(got, a[cuts[g]:cuts[g + 1]].T), g
        dfree(ins[g])
        dfree(outs[g])
    x = rng.integers(-2**31, 2**31, 1_000_003, dtype=np.int64).astype(np.int32)
    cuts = [0, 1, 500_000, 1_000_003]
    ps = [h2d(np.ascontiguousarray(x[cuts[g]:cuts[g + 1]])) for g in range(k)]
    r = np.zeros(1, np.int64)
    for _ in range(5):
        check(L.b2_reduce_sum_multi(vp(*ps), i64(*[cuts[g + 1] - cuts[g] for g in range(k)]), k, _lib.I32,
                                    r.ctypes.data))
        assert int(r[0]) == int(x.astype(np.int64).sum())
    for p in ps:
        dfree(p)


GROUPS = {"transpose": run_transpose, "multi": run_multi, "transpose_big": run_transpose_big, "reduce": run_reduce, "fused": run_fused, "codegen": run_codegen}

if __name__ == "__main__":
    which = sys.argv[1:] or ["all"]
    rng = np.random.default_rng(7)
    for g in (GROUPS if which == ["all"] else which):
        GROUPS[g](rng)
        print("sanitize-driver", g, "ok", flush=True)
