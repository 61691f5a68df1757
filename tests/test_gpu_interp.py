"""run_program drop-in on the GPU vs the reference interpreter's own outputs
(tests/golden, produced by minigpu.interp.run_program)."""
import numpy as np
import pytest

from conftest import program_text
from oracle import oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def b2():
    import paper_2605_13864_b200 as b2
    return b2


def _prog(b2, name):
    return b2.parse_program(program_text(name), name)


def test_golden_cases_through_run_program(b2, golden):
    for c in golden:
        p = _prog(b2, c["program"])
        if c["kind"] == "transpose":
            H, W = c["shape"]
            a = c["inp"]
            params = [n for n, _ in p.fn("transpose").params]
            if "gpu" in c["program"]:
                inputs = {params[0]: a.reshape(-1).tolist(), params[1]: [0.0] * (H * W), "W": W, "H": H}
            else:
                inputs = {params[0]: b2.Array([H, W], a.reshape(-1).tolist(), c["cell"]),
                          params[1]: b2.Array.alloc([W, H], c["cell"]), "W": W, "H": H}
            ret, outs = b2.run_program(p, "transpose", inputs)
            assert ret is None
            got = outs[params[1]]
            want = c["out"].reshape(-1).tolist()
            assert got == want, c["id"]
            assert all(type(v) is type(w) for v, w in zip(got[:4], want[:4])), c["id"]
        else:
            x = c["inp"]
            ret, outs = b2.run_program(p, "reduce", {"arr": x.tolist(), "N": int(x.size)})
            if "result_int" in c:
                assert isinstance(ret, int) and ret == int(c["result_int"]), c["id"]
            elif "tree" in c["program"]:
                assert isinstance(ret, float)
                assert np.float32(ret).view(np.uint32) == np.uint32(c["result_f32_bits"]), c["id"]
            else:
                exact, absum = oracle.sum_f64(x)
                ref = float(np.uint32(c["result_f32_bits"]).view(np.float32))
                assert isinstance(ret, float) and float(np.float32(ret)) == ret
                tol = oracle.f32_tolerance(x.size, exact, absum)
                assert abs(ret - exact) <= tol, c["id"]
                assert abs(ret - exact) <= oracle.f32_gpu_bound(x.size, exact, absum), c["id"]
                # the GPU and the reference (sequential binary32) differ by at most the
                # reference's own measured error plus the tolerance
                assert abs(ret - ref) <= oracle.ref_consistency_bound(ref, exact, tol), c["id"]
            assert outs["arr"] == x.tolist() or "tree" in c["program"] or "result_int" in c


def test_arrays_are_mutated_in_place(b2):
    p = _prog(b2, "transpose_naive.optc")
    src = b2.Array([3, 5], [float(i) for i in range(15)], "float")
    dst = b2.Array.alloc([5, 3], "float")
    b2.Interp(p).run("transpose", {"in": src, "out": dst, "W": 5, "H": 3})
    assert dst.data == np.arange(15, dtype=np.float32).reshape(3, 5).T.reshape(-1).tolist()


def test_sub_block_transpose_with_larger_arrays(b2):
    # in is 6 x 9, the program reads the 4 x 7 corner; out is 10 x 5 and keeps its
    # unwritten cells uninitialised, exactly as the interpreter leaves them
    p = _prog(b2, "transpose_naive.optc")
    a = np.arange(54, dtype=np.float32).reshape(6, 9)
    src = b2.Array([6, 9], a.reshape(-1).tolist(), "float")
    dst = b2.Array.alloc([10, 5], "float")
    b2.run_program(p, "transpose", {"in": src, "out": dst, "W": 7, "H": 4})
    grid = np.array([np.nan if v is None else v for v in dst.data]).reshape(10, 5)
    assert np.array_equal(grid[:7, :4], a[:4, :7].T)
    assert all(v is None for v in np.array(dst.data, dtype=object).reshape(10, 5)[7:].reshape(-1))
    assert all(v is None for v in np.array(dst.data, dtype=object).reshape(10, 5)[:, 4])


@pytest.mark.parametrize("H,W", [(1024, 1024), (4096, 2048), (1000, 3)])
def test_numpy_backed_arrays_zero_copy(b2, H, W):
    p = _prog(b2, "transpose_naive.optc")
    rng = np.random.default_rng(H + W)
    a = rng.standard_normal((H, W)).astype(np.float32)
    out = np.empty((W, H), dtype=np.float32)
    ret, outs = b2.run_program(p, "transpose", {"in": b2.Array.from_numpy(a),
                                                "out": b2.Array.from_numpy(out), "W": W, "H": H})
    assert outs["out"] is not None and np.shares_memory(outs["out"], out)
    assert np.array_equal(out, a.T)


def test_gpu_form_transpose_large(b2):
    p = _prog(b2, "transpose_gpu.optc")
    a = np.random.default_rng(1).standard_normal((2048, 4096)).astype(np.float32)
    out = np.zeros(a.size, dtype=np.float32)
    b2.run_program(p, "transpose", {"in": a.reshape(-1), "out": b2.Array([out.size], out), "W": 4096, "H": 2048})
    assert np.array_equal(out.reshape(4096, 2048), a.T)


def test_bit_pattern_transposes(b2):
    p = _prog(b2, "transpose_naive_int.optc")
    rng = np.random.default_rng(5)
    for dt in (np.uint16, np.uint64, np.int32):
        a = rng.integers(0, np.iinfo(dt).max, (37, 129), dtype=dt)
        out = np.empty((129, 37), dtype=dt)
        b2.run_program(p, "transpose", {"in": b2.Array.from_numpy(a, "int"),
                                        "out": b2.Array.from_numpy(out, "int"), "W": 129, "H": 37})
        assert np.array_equal(out, a.T)


@pytest.mark.parametrize("n", [1 << 20, (1 << 24) + 5])
def test_int_reduce_large_exact(b2, n):
    p = _prog(b2, "reduce_naive_int.optc")
    x = np.random.default_rng(n).integers(-2**31, 2**31, n, dtype=np.int64).astype(np.int32)
    ret, _ = b2.run_program(p, "reduce", {"arr": b2.Array.from_numpy(x, "int"), "N": n})
    assert ret == oracle.reduce_i32(x)


def test_tree_reduce_2_24_bit_exact(b2):
    p = _prog(b2, "reduce_tree_f32.optc")
    x = np.random.default_rng(9).uniform(-1, 1, 1 << 24).astype(np.float32)
    ret, _ = b2.run_program(p, "reduce", {"arr": b2.Array.from_numpy(x), "N": x.size})
    want, _ = oracle.reduce_f32_tree512(x)
    assert np.float32(ret).view(np.uint32) == np.float32(want).view(np.uint32)


def test_naive_f32_reduce_c2(b2):
    p = _prog(b2, "reduce_naive_f32.optc")
    x = np.random.default_rng(2).uniform(-1, 1, 1 << 24).astype(np.float32)
    ret, _ = b2.run_program(p, "reduce", {"arr": b2.Array.from_numpy(x), "N": x.size})
    exact, absum = oracle.sum_f64(x)
    assert abs(ret - exact) <= oracle.f32_tolerance(x.size, exact, absum)


def test_reference_edge_inputs_that_succeed(b2):
    """The edge inputs of tests/golden/ref_interp_errors.json on which the reference
    does NOT raise (e.g. freed host arrays passed to the GPU forms, which only touch
    them through memcpy): same return value here."""
    import json
    import os
    from conftest import GOLDEN
    with open(os.path.join(GOLDEN, "ref_interp_errors.json")) as f:
        cases = [c for c in json.load(f) if c["error"] is None]
    assert len(cases) >= 3
    for c in cases:
        inputs = {k: (b2.Array(list(v["dims"]), list(v["data"]), v["ctype"], v["freed"]) if isinstance(v, dict)
                      else v) for k, v in c["inputs"].items()}
        ret, _ = b2.run_program(_prog(b2, c["program"]), c["entry"], inputs)
        assert ret == c["ret"], c["program"]


def test_int64_cells_sum_exactly_beyond_int64(b2):
    """The reference's ints are unbounded: int64 cells sum in 128 bits, so sums far
    beyond the int64 range come back exact (device, host and run_program paths)."""
    import torch
    rng = np.random.default_rng(64)
    x = rng.integers(-2**63, 2**63, 1_000_003, dtype=np.int64)
    want = sum(int(v) for v in x.tolist())
    assert b2.reduce_sum(x) == want
    from paper_2605_13864_b200.ops import int128
    assert int128(b2.reduce_sum(torch.from_numpy(x).cuda())) == want
    big = np.full(1 << 20, 2**62 + 12345, dtype=np.int64)
    assert b2.reduce_sum(big) == (2**62 + 12345) << 20
    ret, _ = b2.run_program(_prog(b2, "reduce_naive_int.optc"), "reduce",
                            {"arr": [2**40, -3, 2**62, 2**62, 2**62], "N": 5})
    assert ret == 2**40 - 3 + 3 * 2**62
    for off in range(3):  # head / tail paths of the 128-bit kernel
        seg = x[off:off + 70_001]
        assert b2.reduce_sum(torch.from_numpy(seg.copy()).cuda()[0:].contiguous()).shape[0] == 2
        assert int128(b2.reduce_sum(torch.from_numpy(x).cuda()[off:off + 70_001])) == \
            sum(int(v) for v in seg.tolist())
