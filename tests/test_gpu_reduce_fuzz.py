"""Randomised sums through every reduction variant (GPU): cell type, length (0 .. 3 M,
ragged), base misalignment, variant and residency are drawn per case. Integer sums
must equal the exact sum (int32 -> int64, int64 -> 128-bit); fp32 / fp64 sums must be
within the north-star tolerance of the exact sum (oracle.f32_tolerance; binary64
accumulation keeps them near 0.5 ulp)."""
import math

import numpy as np
import pytest

from oracle import oracle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("seed", range(8))
def test_random_sums_every_variant(seed):
    import paper_2605_13864_b200 as b2
    from paper_2605_13864_b200 import _lib
    rng = np.random.default_rng(77 + seed)
    for case in range(25):
        kind = ["i32", "f32", "i64", "f64"][rng.integers(4)]
        n = int(rng.choice([0, 1, 3, 4, 7, 100, 4095, 65537, 1 << 20, 3_000_001]))
        off = int(rng.integers(0, 5))
        variant, ctas = int(rng.integers(0, 10)), int(rng.integers(0, 5))
        if kind == "i32":
            h = rng.integers(-2**31, 2**31, n + off, dtype=np.int64).astype(np.int32)
        elif kind == "i64":
            h = rng.integers(-2**62, 2**62, n + off, dtype=np.int64)
        elif kind == "f32":
            h = (rng.standard_normal(n + off) * np.exp2(rng.integers(-20, 20, n + off))).astype(np.float32)
        else:
            h = rng.standard_normal(n + off) * np.exp2(rng.integers(-40, 40, n + off))
        x = torch.from_numpy(h).cuda()[off:]
        _lib.tune("reduce.variant", variant)
        _lib.tune("reduce.ctas_per_sm", ctas)
        try:
            got = b2.reduce_sum(x)
        finally:
            _lib.tune("reduce.variant", 0)
            _lib.tune("reduce.ctas_per_sm", 0)
        tag = (seed, case, kind, n, off, variant, ctas)
        hv = h[off:]
        if kind in ("i32", "i64"):
            want = sum(int(v) for v in hv.tolist()) if kind == "i64" else int(hv.astype(np.int64).sum())
            got_i = b2.ops.int128(got) if kind == "i64" else int(got.item())
            assert got_i == want, tag
        else:
            if kind == "f32":
                exact, absum = oracle.sum_f64(hv)
            else:  # oracle.sum_f64 is the binary32 helper; fp64 cells: exact fsum
                exact, absum = math.fsum(hv.tolist()), float(np.abs(hv).sum())
            g = float(got.item())
            tol = oracle.f32_tolerance(max(n, 1), exact, absum) if kind == "f32" else \
                max(1e-12 * abs(exact), 2 * n * 2.0**-53 * absum)
            assert abs(g - exact) <= tol, tag
