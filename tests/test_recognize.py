"""Recogniser: alpha-equivalence against the hot-path templates."""
import pytest

from conftest import program_text
from paper_2605_13864_b200 import parse_program, recognize
from paper_2605_13864_b200.recognize import UnsupportedProgram

CASES = {
    "transpose_naive.optc": ("transpose", "naive", "float"),
    "transpose_naive_yx.optc": ("transpose", "naive", "float"),
    "transpose_naive_int.optc": ("transpose", "naive", "int"),
    "transpose_gpu.optc": ("transpose", "gpu", "float"),
    "reduce_naive_f32.optc": ("reduce", "naive", "float"),
    "reduce_naive_int.optc": ("reduce", "naive", "int"),
    "reduce_tree_f32.optc": ("reduce", "tree512", "float"),
}


@pytest.mark.parametrize("name", sorted(CASES))
def test_golden_programs_recognised(name):
    p = parse_program(program_text(name))
    plan = recognize(p, p.entry().name)
    assert (plan.kind, plan.form, plan.cell) == CASES[name]


def test_renaming_and_param_order_are_free():
    src = """void t(int rows, float* dst, int cols, float* src) {
        for (int a = 0; a < cols; a++) { for (int b = 0; b < rows; b++) { dst[a][b] = src[b][a]; } }
    }"""
    plan = recognize(parse_program(src), "t")
    assert plan.params == {"in": "src", "out": "dst", "W": "cols", "H": "rows"}


def test_reference_program_objects_accepted():
    from conftest import reference_available
    if not reference_available():
        pytest.skip("reference not present (GPU box)")
    import minigpu.parser as ref
    p = ref.parse_program(program_text("reduce_tree_f32.optc"))
    assert recognize(p, "reduce").form == "tree512"


@pytest.mark.parametrize("src", [
    # a copy, not a transpose
    "void t(float* in, float* out, int W, int H) { for (int x = 0; x < W; x++) { for (int y = 0; y < H; y++) { out[x][y] = in[x][y]; } } }",
    # shifted read
    "float reduce(float* arr, int N) { float sum = 0.; for (int i = 0; i < N; i++) { sum += arr[i + 1]; } return sum; }",
    # nonzero start
    "float reduce(float* arr, int N) { float sum = 0.; for (int i = 1; i < N; i++) { sum += arr[i]; } return sum; }",
    # nonzero initial value
    "int reduce(int* arr, int N) { int sum = 5; for (int i = 0; i < N; i++) { sum += arr[i]; } return sum; }",
    # same name used for two roles (in == out)
    "void t(float* in, float* out, int W, int H) { for (int x = 0; x < W; x++) { for (int y = 0; y < H; y++) { in[x][y] = in[y][x]; } } }",
    # loop bound swapped with a non-parameter
    "void t(float* in, float* out, int W, int H) { for (int x = 0; x < 7; x++) { for (int y = 0; y < H; y++) { out[x][y] = in[y][x]; } } }",
    # parallel mode differs from the template
    "float reduce(float* arr, int N) { float sum = 0.; parallel for (int i = 0; i < N; i++) { sum += arr[i]; } return sum; }",
])
def test_non_hot_path_programs_refused(src):
    p = parse_program(src)
    with pytest.raises(UnsupportedProgram):
        recognize(p, p.entry().name)


def test_tree_with_other_tile_constant_refused():
    src = program_text("reduce_tree_f32.optc").replace("for (int k = 0; k < 8; k++)",
                                                       "for (int k = 0; k < 7; k++)")
    p = parse_program(src)
    with pytest.raises(UnsupportedProgram):
        recognize(p, "reduce")
