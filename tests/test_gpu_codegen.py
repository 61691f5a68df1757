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


@pytest.mark.parametrize("H,W", [(64, 96), (256, 512), (1024, 2048)])
def test_a4_thread_coarsened_bit_exact(b2, H, W):
    """Check-free launches of A.4 run thread-coarsened (128 CUDA threads play the
    program's 512 per block): same bits as the oracle, and as coarsening off."""
    from paper_2605_13864_b200 import _lib, codegen
    p = _prog(b2, "transpose_gpu.optc")
    a = np.random.default_rng(H * W).standard_normal((H, W)).astype(np.float32)
    inp = {"in": a.reshape(-1).tolist(), "out": [0.0] * (H * W), "W": W, "H": H}
    _, got = b2.run_program(p, "transpose", dict(inp), backend="codegen")
    c = codegen.compile_fn(p.fn("transpose"))
    # 512 program threads per block, 4 KB of shared memory: 4 per CUDA thread (128-thread
    # blocks, 16 resident per SM = 2048 threads), below the 32-block cap: no packing
    assert c.kernel_coarsen()[0] == 4 and c.kernel_pack()[0] == 1 and c.kernel_unchecked()[0]
    assert np.array_equal(np.array(got["out"], np.float32), oracle.transpose(a).reshape(-1))
    prev = _lib.tuning("codegen.coarsen")
    for co in (2, 1):
        _lib.tune("codegen.coarsen", co)
        try:
            _, plain = b2.run_program(p, "transpose", dict(inp), backend="codegen")
            assert c.kernel_coarsen()[0] == co
        finally:
            _lib.tune("codegen.coarsen", prev)
        assert plain["out"] == got["out"]


@pytest.mark.parametrize("blocks,co,pk", [(77, 4, 1), (78, 8, 2), (4096, 8, 2)])
def test_a5_thread_coarsened_bit_exact(b2, blocks, co, pk):
    """A.5 (256 program threads, 1 KB of shared memory per block): an even block count
    packs two program blocks per 64-thread CUDA block at 8 program threads per CUDA
    thread (64 program blocks resident per SM); an odd one stays unpacked at 4. Same
    bits as the oracle's tree order and as packing / coarsening off."""
    from paper_2605_13864_b200 import _lib, codegen
    p = _prog(b2, "reduce_tree_f32.optc")
    x = np.random.default_rng(blocks).uniform(-1, 1, 512 * blocks).astype(np.float32)
    ret, _ = b2.run_program(p, "reduce", {"arr": x.tolist(), "N": x.size}, backend="codegen")
    c = codegen.compile_fn(p.fn("reduce"))
    assert (c.kernel_coarsen()[0], c.kernel_pack()[0]) == (co, pk)
    want, _ = oracle.reduce_f32_tree512(x)
    assert np.float32(ret).view(np.uint32) == np.float32(want).view(np.uint32)
    prev = _lib.tuning("codegen.pack")
    _lib.tune("codegen.pack", 1)
    try:
        plain, _ = b2.run_program(p, "reduce", {"arr": x.tolist(), "N": x.size}, backend="codegen")
        assert c.kernel_pack()[0] == 1
    finally:
        _lib.tune("codegen.pack", prev)
    assert np.float32(plain).view(np.uint32) == np.float32(want).view(np.uint32)


def test_packing_refused_for_block_dependent_barriers(b2):
    """A barrier under an `if` on the block index: packed program blocks would disagree
    on reaching it, so the launch stays one program block per CUDA block (still
    coarsened), with the interpreter's results."""
    from paper_2605_13864_b200 import codegen
    src = """void f(float* a, float* r, int N) {
    float* const d = gmem_malloc1<float>(N);
    memcpy_host_to_device1(d, a, N);
    float* const o = gmem_malloc1<float>(N);
    {
        kernel_launch(N / 128, 128, 4 * 128);
        float* const s = __smem_malloc1<float>(128);
        kernel_setup_end();
        thread for (int b = 0; b < N / 128; b++) {
            thread for (int t = 0; t < 128; t++) { s[DMINDEX1(N / 128, b)][t] = d[b * 128 + t]; }
            if (b % 2 == 0) {
                blocksync();
                thread for (int t = 0; t < 128; t++) { o[b * 128 + t] = s[DMINDEX1(N / 128, b)][127 - t]; }
            } else {
                thread for (int t = 0; t < 128; t++) { o[b * 128 + t] = s[DMINDEX1(N / 128, b)][t] * 2.0; }
            }
        }
        kernel_teardown_begin();
        __smem_free1(s, 128);
        kernel_kill();
    }
    memcpy_device_to_host1(r, o, N);
    gmem_free(o);
    gmem_free(d);
}
"""
    p = b2.parse_program(src)
    n = 128 * 64
    x = np.arange(n, dtype=np.float32)
    _, got = b2.run_program(p, "f", {"a": x.tolist(), "r": [0.0] * n, "N": n}, backend="codegen")
    c = codegen.compile_fn(p.fn("f"))
    assert c.kernel_unchecked()[0] and c.kernel_pack()[0] == 1
    blk = x.reshape(-1, 128)
    want = np.where((np.arange(64) % 2 == 0)[:, None], blk[:, ::-1], blk * 2)
    assert np.array_equal(np.array(got["r"], np.float32), want.reshape(-1))


NOT_COARSENABLE = {
    # a barrier inside a block-level thread-for (the interpreter treats it as a no-op)
    "barrier_in_thread_for": "thread for (int t = 0; t < 128; t++) { o[b * 128 + t] = d[b * 128 + t]; blocksync(); }",
    # program threads accumulate into a block-level local
    "block_local_written": "float acc = 0.0; thread for (int t = 0; t < 128; t++) { acc = acc + 1.0; "
                           "o[b * 128 + t] = d[b * 128 + t] + acc; }",
}


@pytest.mark.parametrize("case", sorted(NOT_COARSENABLE))
def test_coarsening_refused_where_unsound(b2, case):
    from paper_2605_13864_b200 import codegen
    src = f"""void f(float* a, float* r, int N) {{
    float* const d = gmem_malloc1<float>(N);
    memcpy_host_to_device1(d, a, N);
    float* const o = gmem_malloc1<float>(N);
    {{
        kernel_launch(N / 128, 128, 0);
        kernel_setup_end();
        thread for (int b = 0; b < N / 128; b++) {{
            {NOT_COARSENABLE[case]}
        }}
        kernel_teardown_begin();
        kernel_kill();
    }}
    memcpy_device_to_host1(r, o, N);
    gmem_free(o);
    gmem_free(d);
}}
"""
    p = b2.parse_program(src)
    n = 128 * 6
    x = np.arange(n, dtype=np.float32)
    b2.run_program(p, "f", {"a": x.tolist(), "r": [0.0] * n, "N": n}, backend="codegen")
    c = codegen.compile_fn(p.fn("f"))
    assert c.kernel_unchecked()[0] and c.kernel_coarsen()[0] == 1


WIDE_INTERMEDIATE = """void f(float* a, float* r, int N) {
    float* const d = gmem_malloc1<float>(N);
    memcpy_host_to_device1(d, a, N);
    float* const o = gmem_malloc1<float>(N);
    {
        kernel_launch(N / 64, 64, 0);
        kernel_setup_end();
        thread for (int b = 0; b < N / 64; b++) {
            thread for (int t = 0; t < 64; t++) {
                o[b * 64 + t] = d[b * 64 + (t * 100000000) / 100000000];
            }
        }
        kernel_teardown_begin();
        kernel_kill();
    }
    memcpy_device_to_host1(r, o, N);
    gmem_free(o);
    gmem_free(d);
}
"""


def test_32bit_index_arithmetic_only_when_proved(b2):
    """Check-free kernels run with 32-bit integer arithmetic only when the launch
    proof bounds every integer expression below 2^31: A.4 qualifies; an index whose
    intermediate t * 10^8 reaches 6.3e9 keeps 64-bit arithmetic (in 32 bits it would
    wrap and read the wrong cell) and still returns the right cells."""
    from paper_2605_13864_b200 import codegen
    p = _prog(b2, "transpose_gpu.optc")
    a = np.random.default_rng(1).standard_normal((64, 96)).astype(np.float32)
    _, got = b2.run_program(p, "transpose", {"in": a.reshape(-1).tolist(), "out": [0.0] * a.size,
                                             "W": 96, "H": 64}, backend="codegen")
    c = codegen.compile_fn(p.fn("transpose"))
    assert c.kernel_ix32()[0] and c.kernel_unchecked()[0]
    assert np.array_equal(np.array(got["out"], np.float32), a.T.reshape(-1))
    q = b2.parse_program(WIDE_INTERMEDIATE)
    n = 64 * 10
    x = np.random.default_rng(2).standard_normal(n).astype(np.float32)
    _, got = b2.run_program(q, "f", {"a": x.tolist(), "r": [0.0] * n, "N": n}, backend="codegen")
    c = codegen.compile_fn(q.fn("f"))
    assert c.kernel_unchecked()[0] and not c.kernel_ix32()[0]
    assert np.array_equal(np.array(got["r"], np.float32), x)


def test_single_float_ops_match_binary64_rounding(b2):
    """Stores of one +, -, * (and +=) of two binary32 values run in binary32 on the
    device; the interpreter computes them in binary64 and rounds at the store
    (interp.py:43-44, 262-270). Bit-for-bit the same over wide exponents, subnormals,
    exact cancellation and overflow to inf; the nested a * b + a keeps binary64."""
    from test_codegen_cpu import F32_OPS
    rng = np.random.default_rng(2024)
    n = 64 * 4096
    mant = rng.uniform(1, 2, n)
    a = (rng.choice([-1, 1], n) * mant * np.exp2(rng.integers(-149, 128, n))).astype(np.float32)
    b = (rng.choice([-1, 1], n) * rng.uniform(1, 2, n) * np.exp2(rng.integers(-149, 128, n))).astype(np.float32)
    b[::7] = -a[::7]                                   # exact cancellation
    b[1::7] = a[1::7] * np.float32(1 + 2**-23)         # near-ties
    a[2::7] = np.float32(3.4028235e38)                 # overflow to inf
    a[3::7] = np.float32(1e-45) * 3                    # subnormals
    r = np.zeros(5 * n, np.float32)
    p = b2.parse_program(F32_OPS)
    b2.run_program(p, "f", {"a": b2.Array.from_numpy(a), "b": b2.Array.from_numpy(b),
                            "r": b2.Array.from_numpy(r), "N": n}, backend="codegen")
    a64, b64 = a.astype(np.float64), b.astype(np.float64)
    with np.errstate(over="ignore"):
        want = np.stack([a64 + b64, a64 - b64, a64 * b64, a64 * b64 + a64, a64 + b64], 1).astype(np.float32)
    assert np.array_equal(r.reshape(n, 5).view(np.uint32), want.view(np.uint32))


PAIR_PROG = """void f(float* a, float* r, int N, int M) {
    float* const d = gmem_malloc1<float>(N);
    memcpy_host_to_device1(d, a, N);
    float* const o = gmem_malloc1<float>(M);
    {
        kernel_launch(M / 64, 64, 0);
        kernel_setup_end();
        thread for (int t = 0; t < M; t++) {
            o[t] = d[2 * t] * d[2 * t + 1];
        }
        kernel_teardown_begin();
        kernel_kill();
    }
    memcpy_device_to_host1(r, o, M);
    gmem_free(o);
    gmem_free(d);
}
"""


@pytest.mark.parametrize("short", [False, True])
def test_paired_loads_bit_exact_and_bounds(b2, short):
    """`d[2t] * d[2t + 1]` runs as one 64-bit load per program thread in the check-free
    instantiation (bit-exact products); with the input one cell short the last pair is
    out of bounds, the proof fails, and the checked kernel raises the reference's error."""
    from paper_2605_13864_b200 import codegen
    p = b2.parse_program(PAIR_PROG)
    m = 64 * 300
    n = 2 * m - (1 if short else 0)
    a = np.random.default_rng(5).standard_normal(n).astype(np.float32)
    r = np.zeros(m, np.float32)
    args = {"a": b2.Array.from_numpy(a), "r": b2.Array.from_numpy(r), "N": n, "M": m}
    if short:
        with pytest.raises(b2.InterpError, match="out of bounds"):
            b2.run_program(p, "f", args, backend="codegen")
        assert not codegen.compile_fn(p.fn("f")).kernel_unchecked()[0]
        return
    b2.run_program(p, "f", args, backend="codegen")
    assert codegen.compile_fn(p.fn("f")).kernel_unchecked()[0]
    want = (a[0::2].astype(np.float64) * a[1::2].astype(np.float64)).astype(np.float32)
    assert np.array_equal(r.view(np.uint32), want.view(np.uint32))
