"""Generated programs with their full-array copies folded into a chunked
copy -> kernel -> copy pipeline (codegen window + libb200k b2_pipe_run, SURVEY
8f rank 2): same bits as the plain program-order execution and as the
reference's outputs, with pinned and pageable host buffers, many chunks, and
windows the planner must refuse or degrade (whole-array footprints)."""
import json
import os
import random

import numpy as np
import pytest

from conftest import GOLDEN, program_text
from oracle import oracle, vinterp

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def b2():
    import paper_2605_13864_b200 as b2
    return b2


@pytest.fixture
def small_steps():
    """Pipeline steps of 4 KiB: even small programs split into many chunks."""
    from paper_2605_13864_b200 import _lib
    old = _lib.tuning("codegen.pipe_kb")
    _lib.tune("codegen.pipe_kb", 4)
    yield
    _lib.tune("codegen.pipe_kb", old)


def _pinned(shape, dt):
    return torch.empty(shape, dtype=dt, pin_memory=True).numpy()


@pytest.mark.parametrize("pinned", [False, True])
@pytest.mark.parametrize("H,W", [(256, 512), (96, 2048), (1024, 96)])
def test_a4_pipelined_bit_exact(b2, small_steps, pinned, H, W):
    from paper_2605_13864_b200 import codegen
    p = b2.parse_program(program_text("transpose_gpu.optc"))
    a = np.random.default_rng(H + W).standard_normal((H, W)).astype(np.float32)
    if pinned:
        src, dst = _pinned((H, W), torch.float32), _pinned((W, H), torch.float32)
        src[...] = a
        dst[...] = 0
    else:
        src, dst = a.copy(), np.zeros((W, H), np.float32)
    b2.run_program(p, "transpose", {"in": b2.Array([H, W], src.reshape(-1), "float"),
                                    "out": b2.Array([W, H], dst.reshape(-1), "float"), "W": W, "H": H},
                   backend="codegen")
    c = codegen.compile_fn(p.fn("transpose"))
    assert c.kernel_piped()[0] >= 2, c.kernel_piped()
    assert np.array_equal(dst.view(np.uint32), oracle.transpose(a).view(np.uint32))


def test_a5_pipelined_bit_exact(b2, small_steps):
    from paper_2605_13864_b200 import codegen
    p = b2.parse_program(program_text("reduce_tree_f32.optc"))
    x = np.random.default_rng(5).uniform(-1, 1, 512 * 300).astype(np.float32)
    ret, _ = b2.run_program(p, "reduce", {"arr": b2.Array([x.size], x, "float"), "N": x.size}, backend="codegen")
    assert codegen.compile_fn(p.fn("reduce")).kernel_piped()[0] >= 2
    want, _ = oracle.reduce_f32_tree512(x)
    assert np.float32(ret).view(np.uint32) == np.float32(want).view(np.uint32)


def test_golden_programs_pipelined(b2, small_steps):
    """The reference-pinned codegen goldens (derived variants incl. a two-kernel
    program) through the pipeline: same bits as minigpu.interp produced."""
    with open(os.path.join(GOLDEN, "manifest_codegen.json")) as f:
        man = json.load(f)
    arrs = np.load(os.path.join(GOLDEN, "golden_codegen.npz"))
    for c in man["cases"]:
        for k in arrs.files:
            if k.startswith(c["id"] + "_"):
                c[k[len(c["id"]) + 1:]] = arrs[k]
        p = b2.parse_program(program_text(c["program"]), c["program"])
        if c["kind"] == "transpose":
            H, W = c["shape"]
            _, outs = b2.run_program(p, "transpose", {"in": c["inp"].reshape(-1).tolist(),
                                                      "out": [0.0] * (H * W), "W": W, "H": H}, backend="codegen")
            assert outs["out"] == c["out"].reshape(-1).tolist(), c["id"]
        else:
            x = c["inp"]
            ret, _ = b2.run_program(p, "reduce", {"arr": x.tolist(), "N": int(x.size)}, backend="codegen")
            if "result_int" in c:
                assert ret == int(c["result_int"]), c["id"]
            else:
                assert np.float32(ret).view(np.uint32) == np.uint32(c["result_f32_bits"]), c["id"]


def test_random_programs_pipelined_vs_reference_semantics(b2, small_steps):
    """The codegen fuzz family (thread-for nests, shared tiles, barriers, branches)
    with pipelining forced on small inputs: bit-exact against the vectorised
    restatement of the reference interpreter, and against the plain execution."""
    from paper_2605_13864_b200 import _lib, codegen
    from test_gpu_codegen_fuzz import _gen
    _lib.tune("codegen.pipe_kb", 1)  # 1-KiB steps: the family's arrays are 0.25-16 KiB
    rng = random.Random(21)
    ran = piped = 0
    while ran < 12:
        src, n = _gen(rng)
        p = b2.parse_program(src)
        x = np.random.default_rng(ran).uniform(-1, 1, n).astype(np.float32)
        inputs = {"a": x.tolist(), "r": [0.0] * n, "N": n}
        try:
            b2.check_kernels(p, "f", inputs)
        except b2.GateError:
            continue
        _, got = b2.run_program(p, "f", dict(inputs), backend="codegen")
        piped += codegen.compile_fn(p.fn("f")).kernel_piped()[0] >= 2
        _, want = vinterp.run_program(p, "f", dict(inputs))
        assert np.array_equal(np.array(got["r"], np.float32).view(np.uint32),
                              np.array(want["r"], np.float32).view(np.uint32)), src
        _lib.tune("codegen.pipe_kb", 0)
        try:
            _, plain = b2.run_program(p, "f", dict(inputs), backend="codegen")
        finally:
            _lib.tune("codegen.pipe_kb", 1)
        assert plain["r"] == got["r"]
        ran += 1
    assert piped >= 4, piped


WHOLE = """void f(float* a, float* r, int N) {
    float* const d = gmem_malloc1<float>(N);
    memcpy_host_to_device1(d, a, N);
    float* const o = gmem_malloc1<float>(N);
    {
        kernel_launch(N / 64, 64, 0);
        kernel_setup_end();
        thread for (int b = 0; b < N / 64; b++) {
            thread for (int t = 0; t < 64; t++) {
                o[b * 64 + t] = d[N - 1 - (b * 64 + t)] + d[t];
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


def test_reversed_and_shared_footprints(b2, small_steps):
    """Chunk b reads d from the END of the array (a descending band) and the first
    64 cells (shared by all chunks): the input plan must copy whatever a chunk needs
    before it runs, whatever the order; outputs are ascending bands."""
    n = 64 * 200
    x = np.random.default_rng(3).uniform(-1, 1, n).astype(np.float32)
    p = b2.parse_program(WHOLE)
    _, got = b2.run_program(p, "f", {"a": x.tolist(), "r": [0.0] * n, "N": n}, backend="codegen")
    want = (x[::-1] + np.tile(x[:64], n // 64)).astype(np.float32)
    assert np.array_equal(np.array(got["r"], np.float32), want)


def test_pipeline_switch_off(b2, small_steps):
    """B2K_CODEGEN_PIPE=0 / codegen.pipe_kb = 0 keep program order (no chunking)."""
    from paper_2605_13864_b200 import _lib, codegen
    p = b2.parse_program(program_text("transpose_gpu.optc"))
    a = np.arange(64 * 96, dtype=np.float32).reshape(64, 96)
    _lib.tune("codegen.pipe_kb", 0)
    try:
        _, outs = b2.run_program(p, "transpose", {"in": a.reshape(-1).tolist(), "out": [0.0] * a.size,
                                                  "W": 96, "H": 64}, backend="codegen")
    finally:
        _lib.tune("codegen.pipe_kb", 4)
    assert codegen.compile_fn(p.fn("transpose")).kernel_piped()[0] == 0
    assert outs["out"] == a.T.reshape(-1).tolist()
