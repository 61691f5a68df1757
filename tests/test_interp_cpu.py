"""Host-side behaviour of the run_program drop-in that needs no GPU: parameter
marshalling and the reference's error behaviour (tests/golden/ref_errors.json,
recorded from minigpu.interp), raised before any device work."""
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN, program_text
from paper_2605_13864_b200 import Array, InterpError, UnsupportedProgram, f32, parse_program, run_program


def prog(name):
    return parse_program(program_text(name), name)


def test_f32_matches_struct_rounding():
    for v in [0.1, 1e-40, 3.4028235e38, -2.5, 1 / 3]:
        assert f32(v) == float(np.float32(v))


def test_array_helpers_mirror_reference():
    a = Array.alloc([2, 3], "float")
    assert a.data == [None] * 6
    a.set([1, 2], 0.1)
    assert a.get([1, 2]) == f32(0.1)
    with pytest.raises(InterpError, match="read of uninitialized cell"):
        a.get([0, 0])
    with pytest.raises(InterpError, match="out of bounds"):
        a.get([2, 0])
    with pytest.raises(InterpError, match="rank mismatch"):
        a.offset([1])


def _ref_errors():
    with open(os.path.join(GOLDEN, "ref_errors.json")) as f:
        return {e["note"]: e for e in json.load(f)}


def test_reference_error_messages_reproduced():
    ref = _ref_errors()
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
        want = ref[note]
        with pytest.raises(InterpError) as ei:
            run_program(prog(pname), entry, inputs)
        assert str(ei.value) == want["error"], note


def test_empty_loops_return_zero_without_device():
    assert run_program(prog("reduce_naive_f32.optc"), "reduce", {"arr": [1.0] * 4, "N": 0})[0] == 0.0
    r, _ = run_program(prog("reduce_naive_int.optc"), "reduce", {"arr": [1, 2, 3], "N": -3})
    assert r == 0 and isinstance(r, int)
    r, outs = run_program(prog("transpose_naive.optc"), "transpose",
                          {"in": Array([0, 0], [], "float"), "out": Array.alloc([0, 0], "float"), "W": 0, "H": 0})
    assert r is None and outs == {"in": [], "out": []}


def test_flat_lists_rejected_for_rank2_transpose():
    with pytest.raises(InterpError, match="rank mismatch"):
        run_program(prog("transpose_naive.optc"), "transpose",
                    {"in": [0.0, 1.0, 2.0, 3.0, 4.0, 5.0], "out": [0.0] * 6, "W": 3, "H": 2})


def test_unrecognised_program_is_refused_not_interpreted():
    p = parse_program("int f(int* a, int n) { int s = 0; for (int i = 0; i < n; i++) { s += a[i] * 2; } return s; }")
    with pytest.raises(UnsupportedProgram, match="no CPU fallback"):
        run_program(p, "f", {"a": [1, 2], "n": 2})


def test_int_cells_outside_64_bits_refused():
    """int32 and int64 cells sum exactly on the device (128-bit accumulation for
    int64); cells the device cannot hold are refused, never wrapped."""
    for big in (2**70, 2**63):
        with pytest.raises(InterpError, match="64-bit range"):
            run_program(prog("reduce_naive_int.optc"), "reduce", {"arr": [big, 1], "N": 2})


def test_float_overflow_matches_struct_pack():
    """f32(1e39) is whatever struct.pack("f") does on this interpreter: an
    OverflowError on older CPythons, +inf on 3.12+ (interp.py:43-44)."""
    import struct
    try:
        want = struct.unpack("f", struct.pack("f", 1e39))[0]
    except OverflowError:
        with pytest.raises(OverflowError):
            run_program(prog("reduce_naive_f32.optc"), "reduce", {"arr": [1e39], "N": 1})
        return
    from paper_2605_13864_b200.interp import _cells
    assert np.isinf(want) and np.isinf(_cells(Array([2], [1e39, 1.0], "float"), 2, "float")[0])


def _materialise(spec):
    return {k: (Array(list(v["dims"]), list(v["data"]), v["ctype"], v["freed"]) if isinstance(v, dict) else v)
            for k, v in spec.items()}


def test_reference_first_error_reproduced():
    """Which error the reference raises FIRST (type and message), for 40 bad / edge
    inputs to the hot-path programs (tests/golden/ref_interp_errors.json) — decided
    before any device work, so this runs without a GPU."""
    with open(os.path.join(GOLDEN, "ref_interp_errors.json")) as f:
        cases = json.load(f)
    assert len(cases) >= 40
    checked = 0
    for c in cases:
        if c["error"] is None:
            continue  # succeeds in the reference: exercised on the GPU (test_gpu_interp.py)
        with pytest.raises(Exception) as ei:
            run_program(prog(c["program"]), c["entry"], _materialise(c["inputs"]))
        assert (type(ei.value).__name__, str(ei.value)) == (c["type"], c["error"]), c
        checked += 1
    assert checked >= 30
