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


# ---------------------------------------------------------------- derivation families
from program_families import reduce_family, transpose_family  # noqa: E402


@pytest.mark.parametrize("T,R", [(8, 2), (16, 16), (32, 4), (32, 32), (64, 8), (64, 16), (128, 8)])
def test_transpose_family_members_recognised(T, R):
    plan = recognize(parse_program(transpose_family(T, R)), "transpose")
    assert (plan.kind, plan.form) == ("transpose", "gpu")
    if (T, R) != (32, 16):
        assert plan.consts == {"T": T, "R": R}


@pytest.mark.parametrize("B,cell", [(2, "float"), (64, "float"), (128, "int"), (256, "float"), (1024, "float"),
                                    (2048, "int"), (512, "int")])
def test_reduce_family_members_recognised(B, cell):
    plan = recognize(parse_program(reduce_family(B, cell)), "reduce")
    assert plan.kind == "reduce" and plan.cell == cell and plan.consts == {"B": B}


def test_family_near_misses_refused():
    """A member with a changed tree level count (wrong association) or a tile
    whose loads and stores disagree is not any family member."""
    src = reduce_family(256, "float").replace("k < 7", "k < 6")
    assert src != reduce_family(256, "float")
    with pytest.raises(UnsupportedProgram):
        recognize(parse_program(src), "reduce")
    src = transpose_family(64, 16).replace("[bx*64 + x] = ", "[bx*64 + x + 1] = ").replace(
        "d_out[bx*64 + j*16 + y][by*64 + x]", "d_out[bx*64 + j*16 + y][by*64 + x + 1]")
    assert src != transpose_family(64, 16)
    with pytest.raises(UnsupportedProgram):
        recognize(parse_program(src), "transpose")


@pytest.mark.parametrize("body", ["sum = sum + arr[i];", "sum = arr[i] + sum;"])
@pytest.mark.parametrize("cell,zero", [("float", "0."), ("float", "0"), ("int", "0")])
def test_spelled_out_accumulation_recognised(body, cell, zero):
    """`sum = sum + arr[i]` / `sum = arr[i] + sum` store exactly what `sum += arr[i]`
    stores (interp.py:259-276; IEEE / int addition commute): same plan."""
    src = (f"{cell} reduce({cell}* arr, int N) {{ {cell} sum = {zero}; "
           f"for (int i = 0; i < N; i++) {{ {body} }} return sum; }}")
    plan = recognize(parse_program(src), "reduce")
    assert (plan.kind, plan.form, plan.cell) == ("reduce", "naive", cell)


def test_spelled_out_accumulation_same_reference_values():
    from conftest import reference_available
    if not reference_available():
        pytest.skip("reference only in the build container")
    import random
    from minigpu.interp import run_program as rrun
    from minigpu.parser import parse_program as rparse
    rng = random.Random(1)
    xs = [rng.uniform(-1, 1) for _ in range(777)]
    vals = set()
    for body in ["sum += arr[i];", "sum = sum + arr[i];", "sum = arr[i] + sum;"]:
        src = f"float reduce(float* arr, int N) {{ float sum = 0.; for (int i = 0; i < N; i++) {{ {body} }} return sum; }}"
        vals.add(rrun(rparse(src), "reduce", {"arr": xs, "N": len(xs)})[0])
    assert len(vals) == 1
