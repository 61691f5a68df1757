"""Parity at BASELINE.json's full sizes through size-independent properties:
C4 (fp32 32768^2 transpose): involution and row-sum / column-sum checksums on the
bit patterns; C3 (int32 2^30 sum): exact against an independent device sum, the
CPU oracle on the full array, and linearity over random splits; plus the 2^32
end of the C5 sweep."""
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
    # and a sampled tile against the CPU oracle
    r0, c0 = 12345, 23456
    blk = bits[r0:r0 + 64, c0:c0 + 96].cpu().numpy()
    assert np.array_equal(t.view(torch.int32)[c0:c0 + 96, r0:r0 + 64].cpu().numpy(), oracle.transpose(blk))


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
    r0, c0 = rows - 77, cols - 91
    blk = bits[r0:, c0:].cpu().numpy()
    assert np.array_equal(t[c0:, r0:].cpu().numpy(), oracle.transpose(blk))
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
