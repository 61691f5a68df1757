"""Pre-dispatch gate (paper_2605_13864_b200/gate.py): the
reference checker's device-side rules (E-THREADS-CTX, E-DESYNC) decided for the
concrete launch, and the `check=` hook of run_program (which also accepts the
reference's own minigpu.checker.check_program)."""
import numpy as np
import pytest

import paper_2605_13864_b200 as b2
from conftest import program_text, reference_available
from paper_2605_13864_b200 import GateError, check_kernels, parse_program, programs
from program_families import reduce_family, transpose_family


def _tin(H, W):
    return {"in": [0.0] * (H * W), "out": [0.0] * (H * W), "W": W, "H": H}


def _rin(n, v=0.0):
    return {"arr": [v] * n, "N": n}


@pytest.mark.parametrize("T,R", [(8, 2), (16, 16), (32, 4), (32, 32), (64, 8), (64, 16)])
def test_transpose_family_passes(T, R):
    rep = check_kernels(parse_program(transpose_family(T, R)), "transpose", _tin(4 * T, 6 * T))
    assert rep == {"kernels": 1, "blocks": 24}


@pytest.mark.parametrize("B,cell", [(64, "float"), (128, "int"), (256, "float"), (1024, "float"), (2048, "int")])
def test_reduce_family_passes(B, cell):
    rep = check_kernels(parse_program(reduce_family(B, cell)), "reduce", _rin(B * 70, 0))
    assert rep["kernels"] == 1 and rep["blocks"] == 1  # 70 blocks > MAX_BLOCKS: one symbolic pass


def test_canonical_programs_pass():
    assert check_kernels(parse_program(programs.TRANSPOSE_GPU), "transpose", _tin(64, 96))["blocks"] == 6
    assert check_kernels(parse_program(programs.REDUCE_TREE), "reduce", _rin(512 * 9))["blocks"] == 9
    # naive programs have no kernel: nothing to gate
    assert check_kernels(parse_program(programs.TRANSPOSE_NAIVE), "transpose", _tin(8, 8))["kernels"] == 0


def test_wide_context_global_access_is_refused():
    """scale_then_reduce's second kernel reads global memory from a 32-thread
    context (one block-wide statement) — the checker's rule rejects that."""
    with pytest.raises(GateError) as ei:
        check_kernels(parse_program(program_text("scale_then_reduce.optc")), "reduce", _rin(4096))
    assert ei.value.code == "E-THREADS-CTX" and "width 32" in ei.value.message


def test_missing_barrier_in_transpose_is_a_desync():
    src = programs.TRANSPOSE_GPU.replace("blocksync();", "", 1)
    with pytest.raises(GateError) as ei:
        check_kernels(parse_program(src), "transpose", _tin(64, 64))
    assert ei.value.code == "E-DESYNC" and "'tile'" in ei.value.message


def test_missing_barrier_in_tree_level_is_a_desync():
    lines = reduce_family(64, "float").split("\n")
    del lines[[k for k, ln in enumerate(lines) if "blocksync" in ln][1]]
    with pytest.raises(GateError) as ei:
        check_kernels(parse_program("\n".join(lines)), "reduce", _rin(256))
    assert ei.value.code == "E-DESYNC" and "'s'" in ei.value.message


def test_barrier_inside_thread_loop_is_refused():
    src = programs.TRANSPOSE_GPU.replace(
        "tile[DMINDEX2(H/32, W/32, by, bx)][j*16 + y][x] = d_in[by*32 + j*16 + y][bx*32 + x];",
        "tile[DMINDEX2(H/32, W/32, by, bx)][j*16 + y][x] = d_in[by*32 + j*16 + y][bx*32 + x];\n blocksync();", 1)
    with pytest.raises(GateError) as ei:
        check_kernels(parse_program(src), "transpose", _tin(32, 32))
    assert ei.value.code == "E-THREADS-CTX" and "block-wide ThreadsCtx of 512" in ei.value.message


def test_global_write_collision_is_a_desync():
    src = programs.TRANSPOSE_GPU.replace("d_out[bx*32 + j*16 + y][by*32 + x] =", "d_out[bx*32 + j*16 + y][by*32] =", 1)
    with pytest.raises(GateError) as ei:
        check_kernels(parse_program(src), "transpose", _tin(64, 64))
    assert ei.value.code == "E-DESYNC" and "global memory" in ei.value.message


def test_data_dependent_index_is_not_waved_through():
    src = """void f(int* a, int N) {
    int* const d = gmem_malloc1<int>(N);
    memcpy_host_to_device1(d, a, N);
    {
        kernel_launch(1, N, 0);
        kernel_setup_end();
        thread for (int t = 0; t < N; t++) { d[d[t]] = t; }
        kernel_teardown_begin();
        kernel_kill();
    }
    memcpy_device_to_host1(a, d, N);
    gmem_free(d);
}"""
    with pytest.raises(GateError) as ei:
        check_kernels(parse_program(src), "f", {"a": [0] * 8, "N": 8})
    assert ei.value.code == "E-GATE-DATA"


def test_run_program_gate_refuses_before_dispatch():
    """A refused program never reaches the device (this runs without a GPU)."""
    src = programs.TRANSPOSE_GPU.replace("blocksync();", "", 1)
    with pytest.raises(GateError):
        b2.run_program(parse_program(src), "transpose", _tin(64, 64), check="kernels")
    seen = []

    def refuse(prog):
        seen.append(prog)
        raise RuntimeError("no proof")
    with pytest.raises(RuntimeError, match="no proof"):
        b2.run_program(parse_program(programs.TRANSPOSE_GPU), "transpose", _tin(64, 64), check=refuse)
    assert len(seen) == 1
    with pytest.raises(ValueError):
        b2.run_program(parse_program(programs.TRANSPOSE_GPU), "transpose", _tin(64, 64), check="proof")


@pytest.mark.skipif(not reference_available(), reason="reference checker only in the build container")
def test_reference_checker_as_gate():
    """check=minigpu.checker.check_program: the unannotated GPU form carries no
    proof, so the reference's checker refuses it (E-NOMATCH, HostCtx required)
    before anything is dispatched; the annotated naive programs check OK."""
    from minigpu.checker import check_program
    from minigpu.errors import CheckError
    from minigpu.parser import parse_program as rparse
    with pytest.raises(CheckError) as ei:
        b2.run_program(rparse(program_text("transpose_gpu.optc")), "transpose", _tin(64, 64), check=check_program)
    assert ei.value.code == "E-NOMATCH"
    check_program(rparse(program_text("transpose_naive.optc")))  # what the gate would let through


@pytest.mark.gpu
def test_gated_programs_run_on_gpu():
    rng = np.random.default_rng(3)
    a = rng.standard_normal((64, 96)).astype(np.float32)
    _, outs = b2.run_program(parse_program(programs.TRANSPOSE_GPU), "transpose",
                             {"in": a.reshape(-1).tolist(), "out": [0.0] * a.size, "W": 96, "H": 64},
                             check="kernels")
    assert outs["out"] == a.T.reshape(-1).tolist()
    x = rng.integers(-2**31, 2**31, 128 * 40, dtype=np.int64).astype(np.int32)
    ret, _ = b2.run_program(parse_program(reduce_family(128, "int")), "reduce", {"arr": x.tolist(), "N": x.size},
                            check="kernels", backend="codegen")
    assert ret == int(x.astype(np.int64).sum())


def test_assigned_cell_in_index_is_not_tracked():
    """A cell assigned inside the kernel (here in a nested block) may hold any
    value afterwards: indexing with it is refused, never analysed with a stale value."""
    src = """void f(int* a, int N) {
    int* const d = gmem_malloc1<int>(N);
    memcpy_host_to_device1(d, a, N);
    {
        kernel_launch(1, N, 0);
        kernel_setup_end();
        thread for (int t = 0; t < N; t++) { int k = t; { k = 0; } d[k] = t; }
        kernel_teardown_begin();
        kernel_kill();
    }
    memcpy_device_to_host1(a, d, N);
    gmem_free(d);
}"""
    with pytest.raises(GateError) as ei:
        check_kernels(parse_program(src), "f", {"a": [0] * 8, "N": 8})
    assert ei.value.code == "E-GATE-DATA"


@pytest.mark.parametrize("smem,code,msg", [(4 * 32 * 32, None, None),
                                           (4 * 32 * 32 - 4, "E-SMEM", "over-allocation"),
                                           (4 * 32 * 32 + 64, "E-SMEM", "64 bytes left")])
def test_shared_memory_accounting(smem, code, msg):
    """SPEC acceptance 5: over-allocation refused at the malloc, under-allocation
    at kernel_setup_end, the exact size accepted."""
    src = programs.TRANSPOSE_GPU.replace("4 * 32 * 32", str(smem), 1)
    if code is None:
        assert check_kernels(parse_program(src), "transpose", _tin(32, 32))["kernels"] == 1
        return
    with pytest.raises(GateError) as ei:
        check_kernels(parse_program(src), "transpose", _tin(32, 32))
    assert ei.value.code == code and msg in ei.value.message


def test_barrier_flip_block_level_accepted():
    """SPEC acceptance 3: the same barrier at block level (the canonical A.4) is
    accepted; inside the thread loop it is refused (test above)."""
    assert check_kernels(parse_program(programs.TRANSPOSE_GPU), "transpose", _tin(32, 32))["kernels"] == 1


# ---------------------------------------------------------------- large launches
# (> MAX_BLOCKS blocks: one pass with the block indices symbolic)

def test_large_transpose_launch_is_proved_for_every_block():
    # 8192^2 A.4: 65536 blocks, one symbolic pass, tiles of d_out provably disjoint
    rep = check_kernels(parse_program(programs.TRANSPOSE_GPU), "transpose",
                        {"in": np.zeros(8192 * 8192, np.float32), "out": np.zeros(8192 * 8192, np.float32),
                         "W": 8192, "H": 8192})
    assert rep == {"kernels": 1, "blocks": 1}


def _one_kernel(index_expr, n_blocks=100, write=True):
    body = f"o[{index_expr}] = d[b * 32 + t];" if write else f"o[b * 32 + t] = d[{index_expr}];"
    return f"""void f(float* a, float* r, int N) {{
    float* const d = gmem_malloc1<float>(N);
    memcpy_host_to_device1(d, a, N);
    float* const o = gmem_malloc1<float>(N);
    {{
        kernel_launch({n_blocks}, 32, 0);
        kernel_setup_end();
        thread for (int b = 0; b < {n_blocks}; b++) {{
            thread for (int t = 0; t < 32; t++) {{
                {body}
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


def _run_gate(src, n=100 * 32):
    return check_kernels(parse_program(src), "f", {"a": [0.0] * n, "r": [0.0] * n, "N": n})


def test_large_launch_refuses_non_affine_block_index():
    # `b % 7` would alias blocks 0 and 7 — sampling first / second / last block never saw it
    with pytest.raises(GateError) as ei:
        _run_gate(_one_kernel("(b % 7) * 32 + t"))
    assert ei.value.code == "E-GATE-UNSUPPORTED" and "non-affinely" in ei.value.message


def test_large_launch_refuses_overlapping_block_footprints():
    # stride 16 < per-block span 31: blocks b and b + 1 write the same cells
    with pytest.raises(GateError) as ei:
        _run_gate(_one_kernel("b * 16 + t"))
    assert ei.value.code == "E-GATE-UNSUPPORTED" and "disjoint" in ei.value.message
    # the same program with <= MAX_BLOCKS blocks: every block analysed, a real E-DESYNC
    with pytest.raises(GateError) as ei:
        _run_gate(_one_kernel("b * 16 + t", n_blocks=50), n=50 * 32)
    assert ei.value.code == "E-DESYNC"


def test_large_launch_accepts_disjoint_and_read_only_patterns():
    assert _run_gate(_one_kernel("b * 32 + (31 - t)"))["blocks"] == 1  # reversed inside the tile
    assert _run_gate(_one_kernel("(99 - b) * 32 + t"))["blocks"] == 1  # negative block coefficient
    # reads may overlap freely between blocks (only written arrays need disjointness)
    assert _run_gate(_one_kernel("b * 16 + t", write=False))["blocks"] == 1


def test_pointer_offset_rule_aliases_in_the_gate():
    """a[k][j] on a 1-D array is a[k + j] (interp.py:239-240): even thread t writes
    o[t][1] and odd thread t + 1 writes o[t + 1][0], the same cell t + 1."""
    src = """void f(float* a, float* r, int N) {
    float* const o = gmem_malloc1<float>(N);
    {
        kernel_launch(1, 32, 0);
        kernel_setup_end();
        thread for (int t = 0; t < 32; t++) {
            if (t % 2 == 0) { o[t][1] = 1.0; } else { o[t][0] = 2.0; }
        }
        kernel_teardown_begin();
        kernel_kill();
    }
    memcpy_device_to_host1(r, o, N);
    gmem_free(o);
}
"""
    with pytest.raises(GateError) as ei:
        check_kernels(parse_program(src), "f", {"a": [0.0] * 64, "r": [0.0] * 64, "N": 64})
    assert ei.value.code == "E-DESYNC"
