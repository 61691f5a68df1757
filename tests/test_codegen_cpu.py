"""Code generator on the CPU side: every GPU-form fixture
program translates to CUDA C++ that nvcc compiles for sm_100a; programs that are
not GPU programs, or use constructs outside the generator, are refused."""
import shutil

import pytest

from conftest import program_text
from paper_2605_13864_b200 import codegen, parse_program
from paper_2605_13864_b200.errors import UnsupportedProgram

GPU_FORM = ["transpose_gpu.optc", "transpose_gpu_t64.optc", "reduce_tree_f32.optc",
            "reduce_tree_int256.optc", "scale_then_reduce.optc", "oob_kernel.optc"]


def _fn(name):
    p = parse_program(program_text(name), name)
    return p.entry()


@pytest.mark.parametrize("name", GPU_FORM)
def test_generate_structure(name):
    src = codegen.generate(_fn(name))
    assert "__global__ void b2g_kernel0" in src
    assert 'extern "C" int b2g_main' in src
    assert "DMINDEX" not in src
    if "tree" in name or "transpose" in name:
        assert "__syncthreads();" in src and "extern __shared__" in src


@pytest.mark.skipif(shutil.which("nvcc") is None and not __import__("os").path.exists("/usr/local/cuda/bin/nvcc"),
                    reason="nvcc not available")
@pytest.mark.parametrize("name", GPU_FORM)
def test_generated_code_compiles_for_sm100a(name):
    c = codegen.compile_fn(_fn(name))
    assert c.path.endswith(".so")
    assert hasattr(c.lib, "b2g_main")


def test_naive_programs_are_not_gpu_programs():
    for name in ["transpose_naive.optc", "reduce_naive_f32.optc"]:
        with pytest.raises(UnsupportedProgram, match="not a GPU program"):
            codegen.generate(_fn(name))


@pytest.mark.parametrize("src,msg", [
    ("void f(float* a, int n) { float* const d = gmem_malloc1<float>(n); { kernel_launch(1, 32, 0); "
     "kernel_setup_end(); thread for (int t = 0; t < 32; t++) { g(t); } kernel_teardown_begin(); kernel_kill(); } }",
     "inside a kernel"),
    ("void f(float* a, int n) { { kernel_launch(1, 32, 0); kernel_setup_end(); "
     "thread for (int t = 0; t < 32; t++) { a[t] = 1.0; } kernel_teardown_begin(); kernel_kill(); } }",
     "host array"),
    ("void f(float* a, int n) { { kernel_launch(1, 32, 0); kernel_setup_end(); kernel_teardown_begin(); } }",
     "kernel_kill"),
])
def test_unsupported_constructs_refused(src, msg):
    fn = parse_program(src).entry()
    with pytest.raises(UnsupportedProgram, match=msg):
        codegen.generate(fn)


def test_a4_structure_like_spec_acceptance_1():
    """SPEC.md:524 (acceptance 1) asks the emitted transpose to have one
    __global__ function, one shared tile, exactly one __syncthreads(), a launch of
    (W/32)*(H/32) blocks, no DMINDEX / ghosts, and host code with two device
    allocations, one copy each way and two frees. Same checks on our generator's
    output (its runtime calls stand for cudaMalloc / cudaMemcpy / cudaFree)."""
    src = codegen.generate(_fn("transpose_gpu.optc"))
    kernel = src[src.index("__global__"):src.index('extern "C" int b2g_main')]
    host = src[src.index('extern "C" int b2g_main'):]
    assert src.count("__global__") == 1
    assert kernel.count("__syncthreads();") == 1
    assert kernel.count("float *v_tile = (float *)(b2_smem") == 1
    assert "DMINDEX" not in src and "__ghost" not in src
    # the launch: the checked instantiation, or the check-free one when the host
    # proved every access in bounds for the concrete launch — in program order
    # between the copies (twice: the plain path and the pipeline's fallback), plus the
    # chunk launch of the copy / kernel pipeline on its stream
    # (check-free launches also come thread-coarsened — 1, 2 or 4 program threads per
    # CUDA thread — and in 32-bit index arithmetic when the proof bounds every integer)
    sites = 3  # the plain path, the pipeline branch's fallback, the pipeline's chunk launch
    # (and with several small program blocks packed into one CUDA block: B2PK)
    assert host.count("<true, 1, 1, int64_t><<<") == sites
    variants = {"int32_t": ((1, 1), (2, 1), (4, 1), (4, 2), (8, 2)),
                "int64_t": ((1, 1), (2, 1), (4, 1))}
    for ity, vs in variants.items():
        for c, pk in vs:
            assert host.count(f"<false, {c}, {pk}, {ity}><<<") == sites, (c, pk, ity)
    assert host.count("<<<") == 9 * sites
    assert "template <bool B2CK, int B2CO, int B2PK, typename B2IX>" in src and "b2_k < B2CO" in kernel
    assert "b2_k * b2_pbw" in kernel and "%%dynamic_smem_size" in kernel
    assert host.count("b2_run_plan(") == 1 and host.count("b2fp_acc(_fp, 0, 0,") == 2  # d_in read, 2 dims
    assert host.count("b2fp_acc(_fp, 1, 1,") == 2  # d_out written, 2 dims
    assert host.count("b2i_in(") >= 4 and "catch (B2NoProof &)" in host
    assert "b2_exact_div_h(v_W, ((int64_t)32LL)) * b2_exact_div_h(v_H, ((int64_t)32LL))" in host
    assert "(((int64_t)16LL) * ((int64_t)32LL))" in host  # 512 threads per block
    assert host.count("b2_dev_alloc<float>(") == 2
    # (plain path, the pipeline branch's fallback, and its empty-grid case)
    assert host.count("b2_h2d(") == 3 and host.count("b2_d2h(") == 3
    assert host.count(".freed = true;") == 2


def test_a5_structure_tree_loop_with_barrier():
    """SPEC.md:525 (acceptance 2): the reduction kernel holds a sequential halving
    loop with __syncthreads() inside it."""
    src = codegen.generate(_fn("reduce_tree_f32.optc"))
    kernel = src[src.index("__global__"):src.index('extern "C" int b2g_main')]
    start = kernel.index("for (B2IX v_k")  # the index type of the instantiation
    depth, i = 0, kernel.index("{", start)
    while True:  # the loop body: up to the brace that closes the for
        depth += {"{": 1, "}": -1}.get(kernel[i], 0)
        if depth == 0:
            break
        i += 1
    body = kernel[start:i]
    assert body.count("__syncthreads();") == 1  # one barrier per tree level, inside the loop
    assert kernel.count("__syncthreads();") == 2  # plus the one after the pair loads


def test_many_kernels_stay_inside_the_evidence_arrays():
    """A program with more than 64 kernel scopes (the thread-index suite has 100)
    only records timing / proof evidence for the first 64: no write past the
    64-entry arrays of the generated translation unit."""
    import re
    from program_families import thread_index_nests, thread_index_program
    src = codegen.generate(parse_program(thread_index_program(thread_index_nests(100, seed=9))).fn("idx"))
    assert src.count("__global__ void b2g_kernel") == 100
    idx = [int(m) for m in re.findall(r"b2_kernel_(?:ms|unchecked)\[(\d+)\] =", src)]
    assert idx and max(idx) == 63


def test_launch_uniform_thread_for_levels_are_hoisted():
    """A.4's thread-for levels (extents from H, W and literals under the launch-wide
    context) are all launch-uniform: the check-free instantiation takes their width
    splits from the host (kernel parameters filled by the launch-time proof)."""
    src = codegen.generate(_fn("transpose_gpu.optc"))
    kernel = src[src.index("__global__"):src.index('extern "C" int b2g_main')]
    host = src[src.index('extern "C" int b2g_main'):]
    assert kernel.count("const uint32_t _hp") == 6  # by, bx and two (y, x) pairs
    assert "B2CK ? b2_w0 / (uint32_t)" in kernel
    # six levels, evaluated by the bounds proof of the plain launch path, of the
    # pipelined path, and by the pipeline's per-chunk footprint walk
    assert host.count("_w2 = (uint32_t)(_w /") == 18 and "throw B2NoProof{}" in host
    assert host.count("(_B0 * _tpb") == 1  # only the outermost level (by) is narrowed per chunk


def test_assignment_to_loop_index_refused():
    """the reference raises `'k' is not assignable`
    (interp.py:271-272); the generator used to emit a mutable counter the bounds
    proof still trusted."""
    for loop in ("for", "thread for"):
        src = ("void f(float* a, int N) { float* const d = gmem_malloc1<float>(N); { kernel_launch(1, 1, 0); "
               f"kernel_setup_end(); {loop} (int k = 0; k < 1; k++) {{ k = k + 1000000; d[k] = 1.0; }} "
               "kernel_teardown_begin(); kernel_kill(); } memcpy_device_to_host1(a, d, N); gmem_free(d); }")
        with pytest.raises(UnsupportedProgram, match="'k' is not assignable"):
            codegen.generate(parse_program(src).entry())
    src = ("void f(float* a, int N) { float* const d = gmem_malloc1<float>(N); for (int k = 0; k < 2; k++) "
           "{ k = 3; } { kernel_launch(1, 1, 0); kernel_setup_end(); kernel_teardown_begin(); kernel_kill(); } "
           "gmem_free(d); }")
    with pytest.raises(UnsupportedProgram, match="'k' is not assignable"):
        codegen.generate(parse_program(src).entry())


def test_block_scoped_declarations():
    """A declaration inside a block shadows the outer name only inside the block
    (interp.py:248-249): afterwards the loop index is an int again and the kernel
    still compiles with both bindings."""
    src = ("void f(float* a, int N) { float* const d = gmem_malloc1<float>(N); { kernel_launch(1, 1, 0); "
           "kernel_setup_end(); for (int k = 0; k < 4; k++) { if (N > 0) { float k = 0.5; d[0] = k; } d[k] = 1.0; } "
           "kernel_teardown_begin(); kernel_kill(); } memcpy_device_to_host1(a, d, N); gmem_free(d); }")
    s = codegen.generate(parse_program(src).entry())
    assert "float v_k" in s and "B2IX v_k" in s  # the loop index keeps the index type


F32_OPS = """void f(float* a, float* b, float* r, int N) {
    float* const d_a = gmem_malloc1<float>(N);
    memcpy_host_to_device1(d_a, a, N);
    float* const d_b = gmem_malloc1<float>(N);
    memcpy_host_to_device1(d_b, b, N);
    float* const d_r = gmem_malloc1<float>(5 * N);
    {
        kernel_launch(N / 64, 64, 0);
        kernel_setup_end();
        thread for (int i = 0; i < N; i++) {
            d_r[5 * i] = d_a[i] + d_b[i];
            d_r[5 * i + 1] = d_a[i] - d_b[i];
            d_r[5 * i + 2] = d_a[i] * d_b[i];
            d_r[5 * i + 3] = d_a[i] * d_b[i] + d_a[i];
            float t = d_a[i];
            t += d_b[i];
            d_r[5 * i + 4] = t;
        }
        kernel_teardown_begin();
        kernel_kill();
    }
    memcpy_device_to_host1(r, d_r, 5 * N);
    gmem_free(d_r);
    gmem_free(d_b);
    gmem_free(d_a);
}
"""


def test_single_float_ops_stored_in_binary32():
    """One +, -, * (or +=) of two binary32 values stored into a float computes in
    binary32 (__fadd_rn / __fsub_rn / __fmul_rn: the binary64 result the interpreter
    rounds is the same bits); a nested expression keeps binary64 evaluation."""
    src = codegen.generate(parse_program(F32_OPS).entry())
    kernel = src[src.index("__global__"):src.index('extern "C" int b2g_main')]
    assert kernel.count("__fadd_rn(") == 2 and kernel.count("__fsub_rn(") == 1
    assert kernel.count("__fmul_rn(") == 1  # a*b + a keeps the interpreter's binary64 evaluation
    nested = [ln for ln in kernel.splitlines() if "((double)(((double)(" in ln]
    assert len(nested) == 1 and "__f" not in nested[0]


def test_adjacent_cell_pair_is_one_64_bit_load():
    """A.5's `d_a[b * 512 + 2 * t] + d_a[b * 512 + 2 * t + 1]` (an even index and its
    successor on a 1-D device array) reads both cells with one float2 load in the
    check-free instantiation; an odd-based pair, or one on different arrays, stays scalar."""
    src = codegen.generate(_fn("reduce_tree_f32.optc"))
    assert src.count("*reinterpret_cast<const float2 *>(v_d_a + ") == 1
    # int cells are int64 in device memory: a 128-bit longlong2 pair
    src = codegen.generate(_fn("reduce_tree_int256.optc"))
    assert src.count("*reinterpret_cast<const longlong2 *>(v_d_a + ") == 1
    odd = F32_OPS.replace("d_r[5 * i] = d_a[i] + d_b[i];", "d_r[5 * i] = d_a[2 * i + 1] + d_a[2 * i + 2];")
    odd = odd.replace("kernel_launch(N / 64, 64, 0);", "kernel_launch(N / 128, 64, 0);").replace(
        "thread for (int i = 0; i < N; i++)", "thread for (int i = 0; i < N / 2; i++)")
    assert "float2" not in codegen.generate(parse_program(odd).entry())
