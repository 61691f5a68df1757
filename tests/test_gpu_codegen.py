"""Generated CUDA (codegen.py) vs the reference interpreter's outputs for
GPU-form programs, including derived variants no hand-written kernel covers
(tests/golden/manifest_codegen.json, produced by minigpu.interp.run_program)."""
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN, program_text
from oracle import oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def b2():
    import paper_2605_13864_b200 as b2
    return b2


@pytest.fixture(scope="module")
def gcases():
    with open(os.path.join(GOLDEN, "manifest_codegen.json")) as f:
        man = json.load(f)
    arrs = np.load(os.path.join(GOLDEN, "golden_codegen.npz"))
    for c in man["cases"]:
        for k in arrs.files:
            if k.startswith(c["id"] + "_"):
                c[k[len(c["id"]) + 1:]] = arrs[k]
    return man


def _prog(b2, name):
    return b2.parse_program(program_text(name), name)


def test_codegen_cases_bit_exact(b2, gcases):
    assert len(gcases["cases"]) >= 5
    for c in gcases["cases"]:
        p = _prog(b2, c["program"])
        if c["kind"] == "transpose":
            H, W = c["shape"]
            ret, outs = b2.run_program(p, "transpose", {"in": c["inp"].reshape(-1).tolist(),
                                                        "out": [0.0] * (H * W), "W": W, "H": H},
                                       backend="codegen")
            assert outs["out"] == c["out"].reshape(-1).tolist(), c["id"]
        else:
            x = c["inp"]
            ret, _ = b2.run_program(p, "reduce", {"arr": x.tolist(), "N": int(x.size)}, backend="codegen")
            if "result_int" in c:
                assert isinstance(ret, int) and ret == int(c["result_int"]), c["id"]
            else:
                assert np.float32(ret).view(np.uint32) == np.uint32(c["result_f32_bits"]), c["id"]


def test_codegen_error_messages_match_reference(b2, gcases):
    for e in gcases["errors"]:
        p = _prog(b2, e["program"])
        fn = p.fn(e["entry"])
        inputs = {"oob_kernel.optc": {"arr": [0.5] * 128, "N": 128},
                  "transpose_gpu_t64.optc": {"in": [0.0] * (96 * 64), "out": [0.0] * (96 * 64), "W": 96, "H": 64},
                  "reduce_tree_int256.optc": {"arr": [1] * 300, "N": 300}}[e["program"]]
        with pytest.raises(b2.InterpError) as ei:
            b2.run_program(p, fn.name, inputs, backend="codegen")
        assert str(ei.value) == e["error"], e["note"]


def test_canonical_goldens_through_codegen(b2, golden):
    for c in golden:
        if c["program"] not in ("transpose_gpu.optc", "reduce_tree_f32.optc"):
            continue
        p = _prog(b2, c["program"])
        if c["kind"] == "transpose":
            H, W = c["shape"]
            _, outs = b2.run_program(p, "transpose", {"in": c["inp"].reshape(-1).tolist(),
                                                      "out": [0.0] * (H * W), "W": W, "H": H}, backend="codegen")
            assert outs["out"] == c["out"].reshape(-1).tolist(), c["id"]
        else:
            ret, _ = b2.run_program(p, "reduce", {"arr": c["inp"].tolist(), "N": c["n"]}, backend="codegen")
            assert np.float32(ret).view(np.uint32) == np.uint32(c["result_f32_bits"]), c["id"]


def test_codegen_at_scale_numpy_arrays(b2):
    rng = np.random.default_rng(11)
    x = rng.uniform(-1, 1, 1 << 20).astype(np.float32)
    ret, _ = b2.run_program(_prog(b2, "reduce_tree_f32.optc"), "reduce",
                            {"arr": b2.Array.from_numpy(x), "N": x.size}, backend="codegen")
    want, _ = oracle.reduce_f32_tree512(x)
    assert np.float32(ret).view(np.uint32) == np.float32(want).view(np.uint32)
    a = rng.uniform(-1, 1, (1024, 2048)).astype(np.float32)
    out = np.zeros(a.size, np.float32)
    b2.run_program(_prog(b2, "transpose_gpu_t64.optc"), "transpose",
                   {"in": b2.Array.from_numpy(a.reshape(-1)), "out": b2.Array.from_numpy(out),
                    "W": 2048, "H": 1024}, backend="codegen")
    assert np.array_equal(out.reshape(2048, 1024), a.T)


def test_auto_backend_routes_variants(b2):
    # the 64x64 variant is a member of the A.4 family: "auto" and "kernels" run it on
    # the hand-written transpose; scale_then_reduce is no family member: "auto"
    # compiles it, "kernels" refuses it
    p = _prog(b2, "transpose_gpu_t64.optc")
    a = np.arange(64 * 128, dtype=np.float32)
    for backend in ("auto", "kernels"):
        n0 = b2.launch_count()
        _, outs = b2.run_program(p, "transpose", {"in": a.tolist(), "out": [0.0] * a.size, "W": 128, "H": 64},
                                 backend=backend)
        assert outs["out"] == a.reshape(64, 128).T.reshape(-1).tolist()
        assert b2.launch_count() > n0
    q = _prog(b2, "scale_then_reduce.optc")
    x = np.linspace(-1, 1, 2048, dtype=np.float32)
    ret, _ = b2.run_program(q, "reduce", {"arr": x.tolist(), "N": 2048})
    assert isinstance(ret, float)
    with pytest.raises(b2.UnsupportedProgram):
        b2.run_program(q, "reduce", {"arr": x.tolist(), "N": 2048}, backend="kernels")


def test_bounds_proof_selects_check_free_kernels(b2, monkeypatch):
    """Launch-time bounds proofs (codegen._Proof): the paper's programs and the
    derived variants are proved in bounds for their concrete launches and run the
    check-free instantiation with unchanged results; the out-of-bounds program is
    not proved (its checked kernel reports the reference's error), and
    B2K_CODEGEN_PROVE=0 forces the checked kernels."""
    from paper_2605_13864_b200 import codegen
    rng = np.random.default_rng(5)
    H, W = 256, 192
    a = rng.uniform(-1, 1, (H, W)).astype(np.float32)
    x = rng.uniform(-1, 1, 4096).astype(np.float32)
    xi = rng.integers(-1000, 1000, 4096).tolist()
    cases = [("transpose_gpu.optc", "transpose", lambda: {"in": a.reshape(-1).tolist(), "out": [0.0] * (H * W),
                                                          "W": W, "H": H}),
             ("transpose_gpu_t64.optc", "transpose", lambda: {"in": a.reshape(-1).tolist(), "out": [0.0] * (H * W),
                                                              "W": W, "H": H}),
             ("reduce_tree_f32.optc", "reduce", lambda: {"arr": x.tolist(), "N": x.size}),
             ("reduce_tree_int256.optc", "reduce", lambda: {"arr": xi, "N": len(xi)}),
             ("scale_then_reduce.optc", "reduce", lambda: {"arr": x.tolist(), "N": x.size})]
    for name, entry, inputs in cases:
        p = _prog(b2, name)
        c = codegen.compile_fn(p.fn(entry))
        monkeypatch.setenv("B2K_CODEGEN_PROVE", "1")
        got = b2.run_program(p, entry, inputs(), backend="codegen")
        assert all(c.kernel_unchecked()), name
        monkeypatch.setenv("B2K_CODEGEN_PROVE", "0")
        want = b2.run_program(p, entry, inputs(), backend="codegen")
        assert not any(c.kernel_unchecked()), name
        assert got == want, name
    monkeypatch.setenv("B2K_CODEGEN_PROVE", "1")
    p = _prog(b2, "oob_kernel.optc")
    c = codegen.compile_fn(p.fn("shift"))
    with pytest.raises(b2.InterpError, match="out of bounds"):
        b2.run_program(p, "shift", {"arr": [0.5] * 128, "N": 128}, backend="codegen")
    assert not any(c.kernel_unchecked())
