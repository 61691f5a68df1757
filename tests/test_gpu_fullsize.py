"""Parity at BASELINE.json's full sizes: C4 (fp32 32768^2 transpose) bit-exact
against the CPU oracle on the WHOLE matrix, plus involution and row-sum /
column-sum checksums on the bit patterns; the same full comparisons for the 2-
and 8-byte transposes past 2^31 elements; C3 (int32 2^30 sum) exact against an
independent device sum, the CPU oracle on the full array, and linearity over
random splits; fp32 sums at 2^24 / 2^30 / 2^32 on uniform, wide-exponent and
ill-conditioned (cancelling) data against the compensated binary64 sum."""
import json
import os

import numpy as np
import pytest

from oracle import oracle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def b2():
    import paper_2605_13864_b200 as b2
    return b2


def test_c4_transpose_involution_and_checksums(b2):
    n = 32768
    g = torch.Generator(device="cuda").manual_seed(4)
    bits = torch.randint(-2**31, 2**31, (n, n), device="cuda", dtype=torch.int64, generator=g).to(torch.int32)
    a = bits.view(torch.float32)  # arbitrary bit patterns, NaNs included: the permutation must not care
    t = b2.transpose(a)
    # checksum of checksums: row sums of A are the column sums of A^T (exact in int64)
    assert torch.equal(bits.sum(dim=1, dtype=torch.int64), t.view(torch.int32).sum(dim=0, dtype=torch.int64))
    assert torch.equal(bits.sum(dim=0, dtype=torch.int64), t.view(torch.int32).sum(dim=1, dtype=torch.int64))
    tt = b2.transpose(t)
    assert torch.equal(tt.view(torch.int32), bits)
    del tt
    # the whole 32768^2 result, bit for bit, against the CPU oracle (C restatement of
    # the interpreter's nest, all host threads)
    _full_compare(bits, t.view(torch.int32))


def _full_compare(bits, t):
    """Every cell of the device transpose t against oracle.transpose of the input."""
    want = oracle.transpose(bits.cpu().numpy())
    got = t.cpu().numpy()
    assert got.shape == want.shape and np.array_equal(got, want)


def test_c3_int32_sum_exact_and_linear(b2):
    n = 1 << 30
    g = torch.Generator(device="cuda").manual_seed(3)
    x = torch.randint(-2**31, 2**31, (n,), device="cuda", dtype=torch.int64, generator=g).to(torch.int32)
    got = int(b2.reduce_sum(x).item())
    ref_dev = sum(int(c.sum(dtype=torch.int64).item()) for c in x.split(1 << 27))
    assert got == ref_dev
    assert got == oracle.reduce_i32(x.cpu().numpy())
    rng = np.random.default_rng(0)
    for k in rng.integers(1, n - 1, 4).tolist():
        assert got == int(b2.reduce_sum(x[:k]).item()) + int(b2.reduce_sum(x[k:]).item())


def test_c5_int32_sum_2_32(b2):
    n = 1 << 32
    x = torch.full((n,), -2**31, device="cuda", dtype=torch.int32)  # extreme: sum = -2^63 exactly
    assert int(b2.reduce_sum(x).item()) == -2**63
    x.fill_(2**31 - 1)
    assert int(b2.reduce_sum(x).item()) == (2**31 - 1) * n
    del x
    torch.cuda.empty_cache()


@pytest.mark.parametrize("dt,rows,cols", [
    (torch.int16, 32768, 65536),   # bf16-sized cells, 2^31 elements (32-bit index overflow)
    (torch.int64, 16384, 32768),   # fp64-sized cells, 4 GiB per side
    (torch.int16, 46341, 46343),   # odd pitches past 2^31 elements: the padded scalar tile
])
def test_big_transposes_involution_and_checksums(b2, dt, rows, cols):
    """Transposes past 2^31 elements / 4 GiB for the 2- and 8-byte cell paths:
    checksum of checksums (row sums of A = column sums of A^T, exact in int64),
    involution, and a sampled tile against the CPU oracle."""
    g = torch.Generator(device="cuda").manual_seed(rows + cols)
    info = torch.iinfo(dt)
    bits = torch.randint(info.min, info.max, (rows, cols), device="cuda", dtype=dt, generator=g)
    t = b2.transpose(bits)
    assert torch.equal(bits.sum(dim=1, dtype=torch.int64), t.sum(dim=0, dtype=torch.int64))
    assert torch.equal(bits.sum(dim=0, dtype=torch.int64), t.sum(dim=1, dtype=torch.int64))
    _full_compare(bits, t)
    tt = b2.transpose(t)
    del t
    assert torch.equal(tt, bits)
    del tt, bits
    torch.cuda.empty_cache()


def test_c5_fp32_sum_2_32(b2):
    """fp32 sum at the top of the C5 sweep (16 GiB), within the north-star tolerance
    of an independent float64 device sum (oracle.f32_tolerance)."""
    n = 1 << 32
    g = torch.Generator(device="cuda").manual_seed(32)
    x = torch.empty(n, device="cuda", dtype=torch.float32).uniform_(-1, 1, generator=g)
    got = float(b2.reduce_sum(x).item())
    exact = sum(float(c.sum(dtype=torch.float64).item()) for c in x.split(1 << 28))
    absum = sum(float(c.abs().sum(dtype=torch.float64).item()) for c in x.split(1 << 28))
    assert abs(got - exact) <= oracle.f32_tolerance(n, exact, absum)
    del x
    torch.cuda.empty_cache()


def _log(rec):
    """Achieved-error records (B2K_PARITY_LOG=path.jsonl: tools/gpu_parity.sh ->
    profiles/r02_fp32_parity.jsonl)."""
    path = os.environ.get("B2K_PARITY_LOG")
    if path:
        with open(path, "a") as f:
            f.write(json.dumps(rec) + "\n")


def _fp32_data(kind, n, seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    if kind == "u01":
        return torch.empty(n, device="cuda").uniform_(0, 1, generator=g)
    if kind == "wide":  # gen_golden.py's "wide": normal x 2^k, k in [-20, 20)
        x = torch.randn(n, device="cuda", generator=g)
        x.mul_(torch.exp2(torch.randint(-20, 20, (n,), device="cuda", generator=g).to(torch.float32)))
        return x
    # ill-conditioned: wide-exponent values interleaved with the negation of a rotated
    # copy (sum of the pairs is exactly 0) plus a small uniform component, so the sum is
    # ~1e-7 of sum|x|
    h = n // 2
    v = torch.randn(h, device="cuda", generator=g)
    v.mul_(torch.exp2(torch.randint(-20, 20, (h,), device="cuda", generator=g).to(torch.float32)))
    x = torch.empty(n, device="cuda")
    x[0::2] = v
    x[1::2] = -torch.roll(v, 12345)
    del v
    x.add_(torch.empty(n, device="cuda").uniform_(-1e-3, 1e-3, generator=g))
    return x


@pytest.mark.parametrize("log2n", [24, 30, 32])
@pytest.mark.parametrize("kind", ["u01", "wide", "illcond"])
def test_fp32_sum_conditioning(b2, kind, log2n):
    """fp32 sums beyond U[0,1) / U[-1,1) at the C2 / C3 / C5 sizes.
    The B200 sum accumulates in binary64 and rounds once, so it must sit within
    oracle.f32_gpu_bound (~1 ulp of the binary32 result plus n 2^-53 sum|x|) of the
    compensated binary64 sum of the same cells, far inside the north-star
    tolerance. The achieved errors are logged (B2K_PARITY_LOG)."""
    n = 1 << log2n
    x = _fp32_data(kind, n, 1000 * log2n + len(kind))
    got = float(b2.reduce_sum(x).item())
    xh = x.cpu().numpy()
    del x
    torch.cuda.empty_cache()
    exact, absum = oracle.sum_f64(xh)
    del xh
    tol = oracle.f32_tolerance(n, exact, absum)
    bound = oracle.f32_gpu_bound(n, exact, absum)
    err = abs(got - exact)
    ulp = float(np.spacing(np.float32(abs(exact))))
    _log({"test": "fp32_sum", "kind": kind, "n": n, "exact": exact, "sum_abs": absum, "got": got,
          "abs_err": err, "err_ulps": err / ulp, "gpu_bound": bound, "tolerance": tol,
          "err_over_tol": err / tol})
    assert err <= tol, (kind, n, got, exact, tol)
    assert err <= bound, (kind, n, got, exact, bound)
