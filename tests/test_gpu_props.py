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
