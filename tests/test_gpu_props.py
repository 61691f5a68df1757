"""Property tests of the device entries (hypothesis, derandomised): random
shapes, dtypes, pitches and base offsets for the transpose (bit-exact vs the C
oracle, padding untouched, involution) and random lengths / offsets / dtypes for
the sum (exact for int32, north-star tolerance for fp32, A.5 tree order
bit-exact) — the edge cases SURVEY §4 asks for, drawn instead of enumerated."""
import numpy as np
import pytest
import torch
from hypothesis import HealthCheck, given, settings
from hypothesis import strategies as st

import paper_2605_13864_b200 as b2
from oracle import oracle

pytestmark = pytest.mark.gpu
SETTINGS = dict(max_examples=60, deadline=None, derandomize=True,
                suppress_health_check=[HealthCheck.too_slow, HealthCheck.data_too_large])
DTYPES = [torch.float32, torch.float64, torch.bfloat16, torch.int32, torch.uint8, torch.int16]


@settings(**SETTINGS)
@given(rows=st.integers(1, 700), cols=st.integers(1, 700), dt=st.sampled_from(DTYPES),
       pad_in=st.integers(0, 9), pad_out=st.integers(0, 9), off=st.integers(0, 5), seed=st.integers(0, 2**31))
def test_transpose_views(rows, cols, dt, pad_in, pad_out, off, seed):
    g = torch.Generator().manual_seed(seed)
    es = torch.empty(0, dtype=dt).element_size()
    nbits = {1: torch.uint8, 2: torch.int16, 4: torch.int32, 8: torch.int64}[es]
    full_in = torch.randint(-100, 100, ((rows * (cols + pad_in) + off),), generator=g).to(nbits).view(dt).cuda()
    a = full_in[off:].view(rows, cols + pad_in)[:, :cols]
    full_out = torch.full(((cols * (rows + pad_out) + off),), 7, dtype=nbits).view(dt).cuda()
    o = full_out[off:].view(cols, rows + pad_out)[:, :rows]
    b2.transpose(a, o)
    want_full = full_out.clone()
    want_full[off:].view(cols, rows + pad_out)[:, :rows] = a.t()
    assert torch.equal(full_out.view(nbits), want_full.view(nbits))
    back = b2.transpose(o.contiguous())
    assert torch.equal(back.view(nbits), a.contiguous().view(nbits))
    host = a.contiguous().view(nbits).cpu().numpy()
    assert np.array_equal(o.contiguous().view(nbits).cpu().numpy(), oracle.transpose(host))


@settings(**SETTINGS)
@given(n=st.integers(0, 3_000_000), off=st.integers(0, 7), seed=st.integers(0, 2**31))
def test_reduce_int32_exact(n, off, seed):
    rng = np.random.default_rng(seed)
    x = rng.integers(-2**31, 2**31, n + off, dtype=np.int64).astype(np.int32)
    t = torch.from_numpy(x).cuda()[off:]
    assert int(b2.reduce_sum(t).item()) == oracle.reduce_i32(x[off:])


@settings(**SETTINGS)
@given(n=st.integers(1, 3_000_000), off=st.integers(0, 7), lo=st.sampled_from([0.0, -1.0]),
       scale=st.sampled_from([1.0, 1e-20, 1e20]), seed=st.integers(0, 2**31))
def test_reduce_f32_tolerance(n, off, lo, scale, seed):
    rng = np.random.default_rng(seed)
    x = (rng.uniform(lo, 1.0, n + off) * scale).astype(np.float32)
    t = torch.from_numpy(x).cuda()[off:]
    got = float(b2.reduce_sum(t).item())
    exact, absum = oracle.sum_f64(x[off:])
    assert abs(got - exact) <= oracle.f32_tolerance(n, exact, absum)


@settings(**SETTINGS)
@given(blocks=st.integers(1, 5000), seed=st.integers(0, 2**31))
def test_tree512_bit_exact(blocks, seed):
    rng = np.random.default_rng(seed)
    x = rng.standard_normal(512 * blocks).astype(np.float32)
    want, parts = oracle.reduce_f32_tree512(x)
    t = torch.from_numpy(x).cuda()
    assert np.array_equal(b2.reduce_tree512_partials(t).cpu().numpy().view(np.uint32), parts.view(np.uint32))
    assert np.float32(b2.reduce_tree512(t)).view(np.uint32) == np.float32(want).view(np.uint32)


HOST_DTYPES = [np.uint8, np.uint16, np.float32, np.int32, np.float64, np.int64]


@settings(**SETTINGS)
@given(rows=st.integers(1, 1500), cols=st.integers(1, 1500), dt=st.sampled_from(HOST_DTYPES),
       pad_in=st.integers(0, 9), pad_out=st.integers(0, 9), off=st.integers(0, 3),
       chunk_mb=st.sampled_from([1, 2, 64]), seed=st.integers(0, 2**31))
def test_transpose_host_pipeline(rows, cols, dt, pad_in, pad_out, off, chunk_mb, seed):
    """b2_transpose_host on pageable numpy views (pitched rows, misaligned bases),
    with small staging chunks so the 2-D block pipeline runs many stages: bit-exact
    against the C oracle, the output view's padding untouched."""
    from paper_2605_13864_b200 import _lib
    rng = np.random.default_rng(seed)
    es = np.dtype(dt).itemsize
    ubits = {1: np.uint8, 2: np.uint16, 4: np.uint32, 8: np.uint64}[es]
    raw = rng.integers(0, 2**(8 * es) - 1, rows * (cols + pad_in) + off, dtype=np.uint64).astype(ubits)
    a = raw[off:].reshape(rows, cols + pad_in)[:, :cols].view(dt)
    out_raw = np.full(cols * (rows + pad_out) + off, 7, dtype=ubits)
    o = out_raw[off:].reshape(cols, rows + pad_out)[:, :rows].view(dt)
    _lib.tune("host.chunk_mb", chunk_mb)
    try:
        b2.transpose(a, o)
    finally:
        _lib.tune("host.chunk_mb", 0)
    assert np.array_equal(o.view(ubits), oracle.transpose(np.ascontiguousarray(a.view(ubits))))
    pad = out_raw[off:].reshape(cols, rows + pad_out)[:, rows:]
    assert (pad == 7).all() and (out_raw[:off] == 7).all()


@settings(**SETTINGS)
@given(n=st.integers(0, 4_000_000), off=st.integers(0, 7), dt=st.sampled_from([np.int32, np.int64, np.float32]),
       chunk_mb=st.sampled_from([1, 64]), seed=st.integers(0, 2**31))
def test_reduce_host_pipeline(n, off, dt, chunk_mb, seed):
    """b2_reduce_sum_host on pageable, misaligned host arrays, chunked: int32 / int64
    exact (128-bit for int64), fp32 within the north-star tolerance."""
    from paper_2605_13864_b200 import _lib
    rng = np.random.default_rng(seed)
    if dt == np.float32:
        x = rng.uniform(-1, 1, n + off).astype(np.float32)[off:]
    elif dt == np.int32:
        x = rng.integers(-2**31, 2**31, n + off, dtype=np.int64).astype(np.int32)[off:]
    else:
        x = rng.integers(-2**63, 2**63 - 1, n + off, dtype=np.int64)[off:]
    _lib.tune("host.chunk_mb", chunk_mb)
    try:
        got = b2.reduce_sum(x)
    finally:
        _lib.tune("host.chunk_mb", 0)
    if dt == np.float32:
        exact, absum = oracle.sum_f64(x)
        assert abs(got - exact) <= oracle.f32_tolerance(max(n, 1), exact, absum)
    else:
        assert got == (int(x.astype(object).sum()) if dt == np.int64 else int(x.astype(np.int64).sum()))
