"""The vectorised reference-semantics interpreter (oracle/vinterp.py, SURVEY
§8(f) rank 4) against the reference interpreter's own outputs: the golden
fixtures (tests/golden, produced by minigpu.interp.run_program), the reference's
error messages, crafted programs with loop-carried dependences / races /
reductions / early returns (compared with the live reference when it is
importable, i.e. in the build container), lane-budget chunking, and the C
oracle at larger sizes."""
import hashlib
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN, program_text, reference_available
from oracle import oracle, vinterp
from paper_2605_13864_b200 import Array, parse_program, programs
from program_families import reduce_family, transpose_family


def _prog(name):
    return parse_program(program_text(name), name)


def _transpose_inputs(prog, H, W, a, cell):
    pin, pout = [p for p, _ in prog.fn("transpose").params][:2]
    return {pin: Array([H, W], a.reshape(-1).tolist(), cell), pout: Array.alloc([W, H], cell), "W": W, "H": H}, pout


@pytest.mark.parametrize("budget", [vinterp.LANE_BUDGET, 7])
def test_golden_cases(golden, budget):
    assert len(golden) >= 40
    for c in golden:
        prog = _prog(c["program"])
        if c["kind"] == "transpose":
            H, W = c["shape"]
            a = c["inp"]
            if a.dtype == np.uint64:  # fp64 bit patterns: int64 views (vinterp ints are int64)
                a, want = a.view(np.int64), c["out"].view(np.int64)
            else:
                want = c["out"]
            cell = "int" if c["cell"] == "int" else "float"
            inputs, pout = _transpose_inputs(prog, H, W, a, cell)
            _, outs = vinterp.run_program(prog, "transpose", inputs, lane_budget=budget)
            assert outs[pout] == want.reshape(-1).tolist(), c["id"]
        else:
            x = c["inp"]
            ret, _ = vinterp.run_program(prog, "reduce", {"arr": x.tolist(), "N": int(x.size)},
                                         lane_budget=budget)
            if "result_int" in c:
                assert isinstance(ret, int) and ret == int(c["result_int"]), c["id"]
            else:
                assert np.float32(ret).view(np.uint32) == np.uint32(c["result_f32_bits"]), c["id"]


def test_golden_codegen_programs():
    """The derived GPU-form programs (two kernels, int trees, 64-wide tiles)."""
    with open(os.path.join(GOLDEN, "manifest_codegen.json")) as f:
        man = json.load(f)
    arrs = np.load(os.path.join(GOLDEN, "golden_codegen.npz"))
    for c in man["cases"]:
        prog = _prog(c["program"])
        x = arrs[c["id"] + "_inp"]
        if c["kind"] == "transpose":
            H, W = c["shape"]
            _, outs = vinterp.run_program(prog, "transpose", {"in": x.reshape(-1).tolist(), "out": [0.0] * (H * W),
                                                              "W": W, "H": H})
            assert outs["out"] == arrs[c["id"] + "_out"].reshape(-1).tolist(), c["id"]
        else:
            ret, _ = vinterp.run_program(prog, "reduce", {"arr": x.tolist(), "N": int(x.size)})
            if "result_int" in c:
                assert ret == int(c["result_int"]), c["id"]
            else:
                assert np.float32(ret).view(np.uint32) == np.uint32(c["result_f32_bits"]), c["id"]
    for e in man["errors"]:
        prog = _prog(e["program"])
        if e["entry"] == "shift":
            inputs = {"arr": [0.0] * 128, "N": 128}
        elif e["entry"] == "transpose":
            inputs = {"in": [0.0] * (64 * 96), "out": [0.0] * (64 * 96), "W": 96, "H": 64}
        else:
            inputs = {"arr": [1] * 300, "N": 300}
        with pytest.raises(vinterp.InterpError) as ei:
            vinterp.run_program(prog, e["entry"], inputs)
        assert str(ei.value) == e["error"], e["note"]


def test_reference_error_messages():
    with open(os.path.join(GOLDEN, "ref_errors.json")) as f:
        ref = {e["note"]: e for e in json.load(f)}
    cases = {
        "missing input H": ("transpose_naive.optc", "transpose",
                            {"in": Array([2, 3], [0.0] * 6, "float"), "out": Array.alloc([3, 2], "float"), "W": 3}),
        "W larger than in columns": ("transpose_naive.optc", "transpose",
                                     {"in": Array([2, 3], [0.0] * 6, "float"),
                                      "out": Array.alloc([3, 2], "float"), "W": 4, "H": 2}),
        "uninitialised input cell": ("transpose_naive.optc", "transpose",
                                     {"in": Array([2, 3], [0.0] * 5 + [None], "float"),
                                      "out": Array.alloc([3, 2], "float"), "W": 3, "H": 2}),
        "A.4 with 32 not dividing H": ("transpose_gpu.optc", "transpose",
                                       {"in": [0.0] * (33 * 32), "out": [0.0] * (33 * 32), "W": 32, "H": 33}),
        "A.5 with 512 not dividing N": ("reduce_tree_f32.optc", "reduce", {"arr": [1.0] * 513, "N": 513}),
        "N beyond the array": ("reduce_naive_f32.optc", "reduce", {"arr": [1.0] * 4, "N": 5}),
        "use after free": ("reduce_naive_f32.optc", "reduce",
                           {"arr": Array([4], [1.0] * 4, "float", freed=True), "N": 4}),
    }
    for note, (pname, entry, inputs) in cases.items():
        with pytest.raises(vinterp.InterpError) as ei:
            vinterp.run_program(_prog(pname), entry, inputs)
        assert str(ei.value) == ref[note]["error"], note
    assert vinterp.run_program(_prog("reduce_naive_f32.optc"), "reduce", {"arr": [1.0] * 4, "N": 0})[0] == 0.0
    r, _ = vinterp.run_program(_prog("reduce_naive_int.optc"), "reduce", {"arr": [1, 2, 3], "N": -3})
    assert r == 0 and isinstance(r, int)


# crafted programs: name -> (source, entry, inputs factory)
CRAFTED = {
    "prefix_scan": ("void scan(float* a, int N) { for (int i = 1; i < N; i++) { a[i] = a[i - 1] + a[i]; } }",
                    "scan", lambda A: {"a": [0.1 * k for k in range(50)], "N": 50}),
    "reverse_in_place": ("void rev(int* a, int N) { for (int t = 0; t < N; t++) { a[t] = a[N - 1 - t]; } }",
                         "rev", lambda A: {"a": list(range(40)), "N": 40}),
    "nested_float_reduction": (
        "float f(float* a, int N) { float s = 0.; for (int i = 0; i < N; i++) { for (int j = 0; j < 3; j++) "
        "{ s += a[i] * 0.3 + j; } } return s; }",
        "f", lambda A: {"a": [0.1 * k + 1e-3 * k * k for k in range(100)], "N": 100}),
    "branches": ("int f(int* a, int N) { int c = 0; for (int i = 0; i < N; i++) { int v = a[i]; if (v > 5) "
                 "{ a[i] = v * 2; } else { a[i] = 0 - v; } } return c; }",
                 "f", lambda A: {"a": list(range(20)), "N": 20}),
    "private_cells": ("int f(int* a, int N) { int s = 0; for (int i = 0; i < N; i++) { int t = 0; t += a[i]; "
                      "t += 1; a[i] = t; s += t; } return s; }",
                      "f", lambda A: {"a": list(range(30)), "N": 30}),
    "uninitialised": ("float f(float* a, int N) { float* b = MALLOC1<float>(N); float s = 0.; "
                      "for (int i = 0; i < N; i++) { s += b[i]; } return s; }",
                      "f", lambda A: {"a": [1.0] * 4, "N": 4}),
    "use_after_free": ("void f(float* a, int N) { float* b = MALLOC1<float>(N); free(b); "
                       "for (int i = 0; i < N; i++) { b[i] = 1.0; } }", "f", lambda A: {"a": [1.0] * 4, "N": 4}),
    "out_of_bounds": ("void f(float* a, int N) { for (int i = 0; i < N + 1; i++) { a[i] = 1.0; } }",
                      "f", lambda A: {"a": [1.0] * 4, "N": 4}),
    "rank_mismatch": ("void f(float* a, int N) { for (int i = 0; i < N; i++) { a[i][0] = 1.0; } }",
                      "f", lambda A: {"a": A([2, 2], [1.0] * 4, "float"), "N": 2}),
    "early_return": ("int f(int* a, int N) { for (int i = 0; i < N; i++) { if (a[i] == 7) { return i; } } "
                     "return 0 - 1; }", "f", lambda A: {"a": [3, 5, 7, 9, 7], "N": 5}),
    "user_call": ("void g(float* a, int k) { a[k] = a[k] * 2.0; }\n"
                  "void f(float* a, int N) { for (int i = 0; i < N; i++) { g(a, i); } }",
                  "f", lambda A: {"a": [1.5, 2.5, 3.5], "N": 3}),
    "thread_registers": (
        "float f(float* a, int N) { float s = 0.; { kernel_launch(1, 4, 0); kernel_setup_end(); "
        "thread for (int t = 0; t < 4; t++) { float* r = __treg_malloc1<float>(2); r[t][0] = a[t]; "
        "r[t][1] = a[t] * 2.0; a[t] = r[t][0] + r[t][1]; } kernel_teardown_begin(); kernel_kill(); } "
        "for (int i = 0; i < N; i++) { s += a[i]; } return s; }",
        "f", lambda A: {"a": [1.0, 2.0, 3.0, 4.0], "N": 4}),
    "int_intrinsics": ("void f(int* a, int N) { for (int i = 0; i < N; i++) { a[i] = (a[i] % 7) + "
                       "exact_div(a[i] * 3, 3) + pow2(i % 5) + DMINDEX2(N, 3, i, 2); } }",
                       "f", lambda A: {"a": [5, -9, 14, 100, -1, 0, 33], "N": 7}),
    "inexact_division": ("void f(int* a, int N) { for (int i = 0; i < N; i++) { a[i] = exact_div(a[i], 2); } }",
                         "f", lambda A: {"a": [4, 6, 7, 8], "N": 4}),
    "mixed_int_float": ("float f(float* a, int N) { float s = 0.; for (int i = 0; i < N; i++) "
                        "{ s += a[i] * i + 0.1; } return s; }",
                        "f", lambda A: {"a": [0.3 * k for k in range(64)], "N": 64}),
    "triangular_bounds": ("int f(int* a, int N) { int s = 0; for (int i = 0; i < N; i++) { for (int j = 0; j < i; "
                          "j++) { s += a[j] * i; } } return s; }", "f", lambda A: {"a": list(range(25)), "N": 25}),
    "stencil": ("void f(float* a, float* b, int N) { for (int i = 1; i < N - 1; i++) "
                "{ b[i] = a[i - 1] + a[i] + a[i + 1]; } }",
                "f", lambda A: {"a": [0.5 * k for k in range(16)], "b": A([16], [0.0] * 16, "float"), "N": 16}),
    "racy_thread_for": ("void f(int* a, int N) { { kernel_launch(1, N, 0); kernel_setup_end(); "
                        "thread for (int t = 0; t < N; t++) { a[(t + 1) % N] = a[t] + 1; } "
                        "kernel_teardown_begin(); kernel_kill(); } }", "f", lambda A: {"a": list(range(8)), "N": 8}),
    "float_overflow": ("float f(float* a, int N) { float s = 0.; for (int i = 0; i < N; i++) { s += a[i] * 100000000000000000000.0 * 10000000000.0; } "
                       "return s; }", "f", lambda A: {"a": [3e8, 3e8, 3e8], "N": 3}),
}

EXPECTED = {  # the reference's results (minigpu.interp), for boxes without it: (ret, sha256(repr(arrays))[:16])
    'branches': (0, 'fc445d5cf669b77f'),
    'early_return': (2, '3772b5265294005f'),
    'float_overflow': (float("inf"), '2cd802bc40d1ef87'),  # CPython 3.12+: f32() rounds to inf
    'inexact_division': ('ERR', 'InterpError', 'exact_div(7, 2) is not exact'),
    'int_intrinsics': (None, 'df8a7feda420be40'),
    'mixed_int_float': (25609.603515625, 'f26f99f6a04f8305'),
    'nested_float_reduction': (1041.01513671875, '7ef48b9687135942'),
    'out_of_bounds': ('ERR', 'InterpError', 'index 4 out of bounds 0..4'),
    'prefix_scan': (None, 'c54edb537161fd76'),
    'private_cells': (465, 'eed65b5a0905d43b'),
    'racy_thread_for': (None, '41103aebde1360ac'),
    'rank_mismatch': (None, 'b59ad236cc69c612'),
    'reverse_in_place': (None, '4839600e4b81001b'),
    'stencil': (None, '05117a5e4c19dba6'),
    'thread_registers': ('ERR', 'InterpError', 'index 1 out of bounds 0..1'),
    'triangular_bounds': (42550, 'e8d2f29ccb372c7a'),
    'uninitialised': ('ERR', 'InterpError', 'read of uninitialized cell'),
    'use_after_free': ('ERR', 'InterpError', 'use after free'),
    'user_call': (None, 'e6f52cba8e0c3817'),
}


def _run(mod, name, budget=None):
    src, entry, inp = CRAFTED[name]
    A = mod.Array if mod is not vinterp else Array
    kw = {} if budget is None else {"lane_budget": budget}
    try:
        if mod is vinterp:
            return vinterp.run_program(parse_program(src), entry, inp(A), **kw)
        from minigpu.parser import parse_program as rparse
        return mod.run_program(rparse(src), entry, inp(A))
    except Exception as e:  # noqa: BLE001 - compared by type name and message
        return ("ERR", type(e).__name__, str(e))


@pytest.mark.parametrize("name", sorted(CRAFTED))
@pytest.mark.parametrize("budget", [None, 3])
def test_crafted_programs_match_reference(name, budget):
    got = _run(vinterp, name, budget)
    want = EXPECTED[name]
    if want[0] == "ERR":
        assert got[0] == "ERR" and got[1:] == want[1:]
    else:
        assert got[0] == want[0] and hashlib.sha256(repr(got[1]).encode()).hexdigest()[:16] == want[1]
    if not reference_available():
        return
    import minigpu.interp as ref
    want = _run(ref, name)
    if want[0] == "ERR" or got[0] == "ERR":
        assert got[1:] == want[1:] or (got[1] == want[1] and got[2] == want[2])
    else:
        assert got == want


@pytest.mark.parametrize("T,R", [(8, 2), (16, 16), (32, 4)])
def test_transpose_family_members(T, R):
    rng = np.random.default_rng(T + R)
    H, W = 3 * T, 5 * T
    a = rng.standard_normal((H, W)).astype(np.float32)
    prog = parse_program(transpose_family(T, R))
    out = np.zeros(H * W, np.float32)
    vinterp.run_program(prog, "transpose", {"in": Array([H, W], a.reshape(-1), "float"),
                                            "out": Array([W, H], out, "float"), "W": W, "H": H})
    assert np.array_equal(out.reshape(W, H), a.T)


@pytest.mark.parametrize("B,cell", [(64, "float"), (128, "int"), (1024, "float")])
def test_reduce_family_members(B, cell):
    from program_families import np_reduce_family
    rng = np.random.default_rng(B)
    n = 9 * B
    x = rng.uniform(-1, 1, n).astype(np.float32) if cell == "float" else \
        rng.integers(-2**31, 2**31, n, dtype=np.int64).astype(np.int32)
    ret, _ = vinterp.run_program(parse_program(reduce_family(B, cell)), "reduce", {"arr": x.tolist(), "N": n})
    want = np_reduce_family(x, B)
    if cell == "float":
        assert np.float32(ret).view(np.uint32) == np.float32(want).view(np.uint32)
    else:
        assert ret == want


def test_scale_against_c_oracle():
    """Sizes the reference interpreter would need minutes for, in seconds."""
    rng = np.random.default_rng(5)
    H, W = 768, 1024
    a = rng.standard_normal((H, W)).astype(np.float32)
    out = np.zeros(H * W, np.float32)
    vinterp.run_program(parse_program(programs.TRANSPOSE_NAIVE), "transpose",
                        {"in": Array([H, W], a.reshape(-1), "float"), "out": Array([W, H], out, "float"),
                         "W": W, "H": H}, as_numpy=True)
    assert np.array_equal(out.reshape(W, H), oracle.transpose(a))
    out2 = np.zeros(H * W, np.float32)
    vinterp.run_program(parse_program(programs.TRANSPOSE_GPU), "transpose",
                        {"in": Array([H, W], a.reshape(-1), "float"), "out": Array([W, H], out2, "float"),
                         "W": W, "H": H}, as_numpy=True)
    assert np.array_equal(out2, out)
    xi = rng.integers(-2**31, 2**31, 1 << 21, dtype=np.int64).astype(np.int32)
    r, _ = vinterp.run_program(parse_program(programs.REDUCE_NAIVE_INT), "reduce",
                               {"arr": Array([xi.size], xi, "int"), "N": xi.size}, as_numpy=True)
    assert r == oracle.reduce_i32(xi)
    xf = rng.uniform(-1, 1, 1 << 20).astype(np.float32)
    r, _ = vinterp.run_program(parse_program(programs.source(programs.REDUCE_NAIVE, "float")), "reduce",
                               {"arr": Array([xf.size], xf, "float"), "N": xf.size}, as_numpy=True)
    assert np.float32(r) == np.float32(oracle.reduce_f32_seq(xf))
    it = vinterp.VInterp(parse_program(programs.REDUCE_TREE))
    r, _ = it.run("reduce", {"arr": Array([xf.size], xf, "float"), "N": xf.size})
    assert np.float32(r[1]) == np.float32(oracle.reduce_f32_tree512(xf)[0])
    assert it.restarts >= 1  # the level loop `for k` carries a dependence: run sequentially
