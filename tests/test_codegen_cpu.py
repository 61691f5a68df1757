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
