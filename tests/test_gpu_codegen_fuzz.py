"""Random GPU-form programs (kernel scopes with thread-for nests, shared-memory
tiles, barriers, sequential loops, branches on thread indices) through the code
generator on the B200, checked bit for bit against the vectorised restatement of
the reference interpreter (oracle/vinterp.py). Programs the gate refuses
(races, misplaced barriers) are dropped first: the generated kernels only
promise the sequential semantics for race-free programs, as the paper's
checker does."""
import random

import numpy as np
import pytest

import paper_2605_13864_b200 as b2
from oracle import vinterp

pytestmark = pytest.mark.gpu
N_PROGRAMS = 16


def _gen(rng):
    T = rng.choice([32, 64, 128, 256])
    B = rng.choice([1, 3, 8])
    K = rng.randint(1, T - 1)
    split = rng.random() < 0.5 and T >= 64
    op = rng.choice(["* 2.0 + 1.0", "- 0.5", "* d[b * T + t]"]).replace("T", str(T))
    perm = rng.choice([f"(t + {K}) % {T}", f"{T - 1} - t", "t", f"(t * 3) % {T}" if T % 3 else "t"])
    body2 = f"o[b * {T} + t] = s[DMINDEX1({B}, b)][{perm}] + s[DMINDEX1({B}, b)][t];"
    if rng.random() < 0.3:
        body2 = f"if (t % 2 == 0) {{ o[b * {T} + t] = s[DMINDEX1({B}, b)][{perm}]; }} else {{ o[b * {T} + t] = 0.25; }}"
    if split:
        Y = 2 if rng.random() < 0.5 else 4
        X = T // Y
        stage1 = (f"thread for (int y = 0; y < {Y}; y++) {{ thread for (int x = 0; x < {X}; x++) {{ "
                  f"s[DMINDEX1({B}, b)][y * {X} + x] = d[b * {T} + y * {X} + x] {op.replace('[b * ' + str(T) + ' + t]', '[b * ' + str(T) + ' + y * ' + str(X) + ' + x]')}; }} }}")
    else:
        stage1 = f"thread for (int t = 0; t < {T}; t++) {{ s[DMINDEX1({B}, b)][t] = d[b * {T} + t] {op}; }}"
    extra = ""
    if rng.random() < 0.4:  # a sequential loop of in-place updates, each thread its own cell
        extra = (f"for (int k = 0; k < 3; k++) {{ thread for (int t = 0; t < {T}; t++) "
                 f"{{ s[DMINDEX1({B}, b)][t] = s[DMINDEX1({B}, b)][t] * 0.5 + k; }} }}")
    barrier2 = "blocksync();" if rng.random() < 0.9 else ""  # sometimes racy: the gate must drop it
    src = f"""void f(float* a, float* r, int N) {{
    float* const d = gmem_malloc1<float>(N);
    memcpy_host_to_device1(d, a, N);
    float* const o = gmem_malloc1<float>(N);
    {{
        kernel_launch({B}, {T}, 4 * {T});
        float* const s = __smem_malloc1<float>({T});
        kernel_setup_end();
        thread for (int b = 0; b < {B}; b++) {{
            {stage1}
            {extra}
            {barrier2}
            thread for (int t = 0; t < {T}; t++) {{ {body2} }}
        }}
        kernel_teardown_begin();
        __smem_free1(s, {T});
        kernel_kill();
    }}
    memcpy_device_to_host1(r, o, N);
    gmem_free(o);
    gmem_free(d);
}}
"""
    return src, B * T


def test_random_gpu_programs_codegen_vs_reference_semantics():
    rng = random.Random(5)
    ran = refused = 0
    while ran < N_PROGRAMS:
        src, n = _gen(rng)
        p = b2.parse_program(src)
        x = np.random.default_rng(ran).uniform(-1, 1, n).astype(np.float32)
        inputs = {"a": x.tolist(), "r": [0.0] * n, "N": n}
        try:
            b2.check_kernels(p, "f", inputs)
        except b2.GateError:
            refused += 1
            continue
        _, got = b2.run_program(p, "f", dict(inputs), backend="codegen")
        _, want = vinterp.run_program(p, "f", dict(inputs))
        assert np.array_equal(np.array(got["r"], np.float32).view(np.uint32),
                              np.array(want["r"], np.float32).view(np.uint32)), src
        ran += 1
    assert refused >= 0


def _gen_bounds(rng):
    """A one-kernel program whose index expressions are sometimes out of bounds
    (offsets, strides, guards, wrapped indices): the launch-time bounds proof must
    never select the check-free kernel for a program the reference rejects."""
    T = rng.choice([32, 64, 128])
    B = rng.choice([1, 2, 5])
    D = rng.choice([0, 0, 1, -1])
    S = rng.choice([1, 1, 2])
    E = rng.choice([0, 0, 3])
    lim = rng.choice([T, T - 1, T // 2, T // S])
    src_ix = f"b * {T} + t * {S} + {E}"
    if rng.random() < 0.3:
        src_ix = f"({src_ix}) % {rng.choice([B * T, B * T + 1, B * T - 1])}"
    # a block-local declaration shadowing the thread index must not narrow the
    # outer `t` for the proof (interval leaked out of the block)
    shadow = f"if (N > 0) {{ int t = {rng.choice([0, 1])}; }}" if rng.random() < 0.4 else ""
    src = f"""void f(float* a, float* r, int N) {{
    float* const d = gmem_malloc1<float>(N);
    memcpy_host_to_device1(d, a, N);
    float* const o = gmem_malloc1<float>(N);
    memcpy_host_to_device1(o, r, N);
    {{
        kernel_launch({B}, {T}, 0);
        kernel_setup_end();
        thread for (int b = 0; b < {B}; b++) {{
            thread for (int t = 0; t < {T}; t++) {{
                {shadow}
                if (t < {lim}) {{ o[b * {T} + t + {D}] = d[{src_ix}] * 2.0; }}
            }}
        }}
        kernel_teardown_begin();
        kernel_kill();
    }}
    memcpy_device_to_host1(r, o, N);
    gmem_free(o);
    gmem_free(d);
}}
"""
    return src, B * T


def test_random_bounds_programs_proof_is_sound():
    from paper_2605_13864_b200 import codegen
    rng = random.Random(11)
    errors = proved = 0
    for i in range(40):
        src, n = _gen_bounds(rng)
        p = b2.parse_program(src)
        x = np.random.default_rng(i).uniform(-1, 1, n).astype(np.float32)
        inputs = {"a": x.tolist(), "r": [0.0] * n, "N": n}
        try:
            _, want = vinterp.run_program(p, "f", dict(inputs))
            ref_err = None
        except Exception as e:  # noqa: BLE001 - the reference's error
            ref_err = e
        c = codegen.compile_fn(p.fn("f"))
        if ref_err is not None:
            with pytest.raises(b2.InterpError, match="out of bounds"):
                b2.run_program(p, "f", dict(inputs), backend="codegen")
            assert not any(c.kernel_unchecked()), src
            errors += 1
        else:
            _, got = b2.run_program(p, "f", dict(inputs), backend="codegen")
            assert np.array_equal(np.array(got["r"], np.float32).view(np.uint32),
                                  np.array(want["r"], np.float32).view(np.uint32)), src
            proved += all(c.kernel_unchecked())
    assert errors >= 5 and proved >= 5, (errors, proved)


SHADOW = """void f(float* a, int N) {
    float* const d = gmem_malloc1<float>(N);
    {
        kernel_launch(1, 1, 0);
        kernel_setup_end();
        for (int k = 0; k < 10; k++) {
            if (N > 0) { int k = 5; d[k] = 2.0; }
            d[k] = 1.0;
        }
        kernel_teardown_begin();
        kernel_kill();
    }
    memcpy_device_to_host1(a, d, N);
    gmem_free(d);
}
"""


def test_shadowing_decl_does_not_fool_the_proof():
    """the inner `int k = 5` used to replace the loop's interval
    for the outer d[k]; with N = 6 the check-free kernel ran and wrote d[6..9]. The
    reference raises `index 6 out of bounds 0..6` (checked in the build container)."""
    from paper_2605_13864_b200 import codegen
    p = b2.parse_program(SHADOW)
    with pytest.raises(b2.InterpError, match=r"index 6 out of bounds"):
        b2.run_program(p, "f", {"a": [0.0] * 6, "N": 6}, backend="codegen")
    assert not any(codegen.compile_fn(p.fn("f")).kernel_unchecked())
    # in bounds (N = 10): proved, and the result is the reference's (minigpu.interp
    # returns d[5] = 2.0: iterations k = 6..9 rewrite it after k = 5 set it to 1.0)
    _, got = b2.run_program(p, "f", {"a": [0.0] * 10, "N": 10}, backend="codegen")
    assert got["a"] == [1.0] * 5 + [2.0] + [1.0] * 4
    assert all(codegen.compile_fn(p.fn("f")).kernel_unchecked())
