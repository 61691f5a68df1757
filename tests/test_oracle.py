"""Pin the CPU oracle (C and numpy restatements) to the reference's own outputs.

The golden vectors were produced by the reference interpreter
(minigpu.interp.run_program, interp.py:380) via tests/golden/gen_golden.py.
"""
import numpy as np
import pytest

from oracle import oracle


def _expected_int(c):
    return int(c["result_int"])


def test_golden_transposes(golden):
    cases = [c for c in golden if c["kind"] == "transpose"]
    assert len(cases) >= 15
    for c in cases:
        a, ref = c["inp"], c["out"]
        assert np.array_equal(oracle.transpose(a), ref), c["id"]
        assert np.array_equal(oracle.transpose(a, nthreads=1), ref), c["id"]
        assert np.array_equal(oracle.np_transpose(a), ref), c["id"]
        assert ref.tobytes() == np.ascontiguousarray(a.T).tobytes()


def test_golden_reductions(golden):
    cases = [c for c in golden if c["kind"] == "reduce"]
    assert len(cases) >= 25
    for c in cases:
        x = c["inp"]
        if "result_int" in c:
            assert oracle.reduce_i32(x) == _expected_int(c), c["id"]
            assert oracle.np_reduce_i32(x) == _expected_int(c), c["id"]
        elif "tree" in c["program"]:
            want = np.uint32(c["result_f32_bits"]).view(np.float32)
            got, parts = oracle.reduce_f32_tree512(x)
            got2, parts2 = oracle.np_reduce_f32_tree512(x)
            assert np.float32(got).view(np.uint32) == want.view(np.uint32), c["id"]
            assert np.float32(got2).view(np.uint32) == want.view(np.uint32), c["id"]
            assert np.array_equal(parts.view(np.uint32), parts2.view(np.uint32))
        else:
            want = np.uint32(c["result_f32_bits"])
            assert np.float32(oracle.reduce_f32_seq(x)).view(np.uint32) == want, c["id"]
            assert np.float32(oracle.np_reduce_f32_seq(x)).view(np.uint32) == want, c["id"]


def test_spec_golden_values(golden):
    # SPEC.md:501 reduce([1..12]) == 78 and SPEC.md:502 8x8 index transpose.
    r = [c for c in golden if c["kind"] == "reduce" and c["n"] == 12]
    assert {c.get("result_int", c.get("result")) for c in r} <= {"78", 78.0}
    t = golden[0]
    assert t["shape"] == [8, 8]
    assert np.array_equal(t["out"], np.arange(64, dtype=np.float32).reshape(8, 8).T)


def test_int_no_wrap(golden):
    c = [c for c in golden if c.get("note") == "4 x INT32_MAX, no wrap"][0]
    assert int(c["result_int"]) == 8589934588 == oracle.reduce_i32(c["inp"])


@pytest.mark.parametrize("n", [0, 1, 511, 4097, 1 << 18])
def test_restatements_agree_random(n):
    rng = np.random.default_rng(n)
    x = rng.uniform(-1, 1, n).astype(np.float32)
    assert np.float32(oracle.reduce_f32_seq(x)) == np.float32(oracle.np_reduce_f32_seq(x))
    xi = rng.integers(-2**31, 2**31, n, dtype=np.int64).astype(np.int32)
    assert oracle.reduce_i32(xi) == oracle.np_reduce_i32(xi) == int(xi.astype(np.int64).sum())
    if n and n % 512 == 0:
        assert oracle.reduce_f32_tree512(x)[0] == oracle.np_reduce_f32_tree512(x)[0]


@pytest.mark.parametrize("shape,dt", [((1023, 1025), np.float32), ((257, 129), np.uint16),
                                      ((65, 33), np.float64), ((1, 1000), np.int32)])
def test_transpose_restatements_agree(shape, dt):
    rng = np.random.default_rng(7)
    a = rng.integers(0, 2**15, shape).astype(dt)
    assert np.array_equal(oracle.transpose(a), a.T)


def test_tree512_rejects_inexact():
    with pytest.raises(ValueError):
        oracle.reduce_f32_tree512(np.ones(513, np.float32))


def test_tolerance_contains_reference_seq(golden):
    # The tolerance bound used for the GPU parity must contain the reference's own
    # sequential-order error at the golden sizes.
    for c in golden:
        if c["kind"] != "reduce" or "result_f32_bits" not in c or "tree" in c["program"]:
            continue
        x = c["inp"]
        exact, absum = oracle.sum_f64(x)
        ref = float(np.uint32(c["result_f32_bits"]).view(np.float32))
        assert abs(ref - exact) <= oracle.f32_seq_error_bound(x.size, absum) + 1e-30
