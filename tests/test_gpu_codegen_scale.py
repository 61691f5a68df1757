"""Generated kernels (codegen.py) at sizes the reference interpreter cannot
reach, checked bit for bit against the vectorised restatement of the reference
interpreter (oracle/vinterp.py, itself pinned to the reference's outputs in
tests/test_vinterp.py) — for derived programs that have no hand-written
numpy restatement, e.g. the two-kernel scale_then_reduce."""
import numpy as np
import pytest

import paper_2605_13864_b200 as b2
from conftest import program_text
from oracle import vinterp
from program_families import reduce_family, transpose_family

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("T,R", [(16, 4), (32, 8), (64, 16)])
def test_transpose_family_vs_vinterp(T, R):
    rng = np.random.default_rng(T * R)
    H, W = 1024, 1536
    a = rng.standard_normal((H, W)).astype(np.float32)
    prog = b2.parse_program(transpose_family(T, R))
    got = np.zeros(H * W, np.float32)
    b2.run_program(prog, "transpose", {"in": b2.Array([H * W], a.reshape(-1), "float"),
                                       "out": b2.Array([H * W], got, "float"), "W": W, "H": H}, backend="codegen")
    want = np.zeros(H * W, np.float32)
    vinterp.run_program(prog, "transpose", {"in": b2.Array([H * W], a.reshape(-1), "float"),
                                            "out": b2.Array([H * W], want, "float"), "W": W, "H": H},
                        as_numpy=True)
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))


@pytest.mark.parametrize("blocks", [2048, 2047])
@pytest.mark.parametrize("B,cell", [(256, "float"), (1024, "float"), (512, "int")])
def test_reduce_family_vs_vinterp(B, cell, blocks):
    """Also the block packing of generated kernels: B = 256 / 512 (128 / 256 program
    threads) pack two program blocks per CUDA block on an even block count, and run
    unpacked on an odd one — the same bits either way."""
    from paper_2605_13864_b200 import codegen
    rng = np.random.default_rng(B + blocks)
    n = B * blocks
    x = rng.uniform(-1, 1, n).astype(np.float32) if cell == "float" else \
        rng.integers(-2**31, 2**31, n, dtype=np.int64).astype(np.int32)
    prog = b2.parse_program(reduce_family(B, cell))
    arr = b2.Array([n], x, cell)
    got, _ = b2.run_program(prog, "reduce", {"arr": arr, "N": n}, backend="codegen")
    c = codegen.compile_fn(prog.fn("reduce"))
    assert c.kernel_pack()[0] == (2 if (B <= 512 and blocks % 2 == 0) else 1), (B, blocks, c.kernel_pack())
    want, _ = vinterp.run_program(prog, "reduce", {"arr": b2.Array([n], x.copy(), cell), "N": n}, as_numpy=True)
    if cell == "float":
        assert np.float32(got).view(np.uint32) == np.float32(want).view(np.uint32)
    else:
        assert got == want


def test_two_kernel_program_vs_vinterp():
    """scale_then_reduce: y = x * 0.1 + 1.5 (binary64 evaluate, binary32 store),
    per-64 block sums, host loop `sum += p[i] * 2.0 - 1.0` — 2^20 elements."""
    rng = np.random.default_rng(9)
    n = 1 << 20
    x = rng.uniform(-1, 1, n).astype(np.float32)
    prog = b2.parse_program(program_text("scale_then_reduce.optc"))
    got, _ = b2.run_program(prog, "reduce", {"arr": b2.Array([n], x.copy(), "float"), "N": n}, backend="codegen")
    want, _ = vinterp.run_program(prog, "reduce", {"arr": b2.Array([n], x.copy(), "float"), "N": n}, as_numpy=True)
    assert np.float32(got).view(np.uint32) == np.float32(want).view(np.uint32)
