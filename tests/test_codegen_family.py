"""Fuzz the code generator over parametrised program families (tile size, rows
per thread, reduction block size, cell type). The families' numpy restatements
are pinned to the reference interpreter (tests/golden/families_pinned.json);
on the GPU every member must match its restatement bit for bit. The CPU half
compiles every member for sm_100a (and warms the build cache the GPU box uses)."""
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN
from program_families import np_reduce_family, reduce_family, transpose_family
from paper_2605_13864_b200 import codegen, parse_program

TRANSPOSES = [(8, 2), (16, 16), (32, 4), (32, 32), (64, 8), (64, 16)]
REDUCES = [(64, "float"), (128, "int"), (256, "float"), (1024, "float"), (2048, "int")]


def test_family_restatements_pinned_to_reference():
    with open(os.path.join(GOLDEN, "families_pinned.json")) as f:
        members = json.load(f)["members"]
    assert len(members) >= 9
    assert all(m.get("ref_equals_transpose", m.get("ref_equals_restatement")) for m in members)


@pytest.mark.parametrize("T,R", TRANSPOSES)
def test_transpose_family_compiles(T, R):
    assert codegen.compile_fn(parse_program(transpose_family(T, R)).entry()).n_kernels == 1


@pytest.mark.parametrize("B,cell", REDUCES)
def test_reduce_family_compiles(B, cell):
    assert codegen.compile_fn(parse_program(reduce_family(B, cell)).entry()).n_kernels == 1


@pytest.mark.gpu
@pytest.mark.parametrize("T,R", TRANSPOSES)
def test_transpose_family_on_gpu(T, R):
    import paper_2605_13864_b200 as b2
    rng = np.random.default_rng(T * 100 + R)
    H, W = 5 * T, 7 * T
    a = rng.standard_normal((H, W)).astype(np.float32)
    out = np.zeros(H * W, np.float32)
    b2.run_program(parse_program(transpose_family(T, R)), "transpose",
                   {"in": b2.Array.from_numpy(a.reshape(-1)), "out": b2.Array.from_numpy(out), "W": W, "H": H},
                   backend="codegen")
    assert np.array_equal(out.reshape(W, H), a.T)


@pytest.mark.gpu
@pytest.mark.parametrize("B,cell", REDUCES)
def test_reduce_family_on_gpu(B, cell):
    import paper_2605_13864_b200 as b2
    rng = np.random.default_rng(B)
    n = 37 * B
    x = rng.uniform(-1, 1, n).astype(np.float32) if cell == "float" else \
        rng.integers(-2**31, 2**31, n, dtype=np.int64).astype(np.int32)
    ret, _ = b2.run_program(parse_program(reduce_family(B, cell)), "reduce",
                            {"arr": x.tolist(), "N": n}, backend="codegen")
    want = np_reduce_family(x, B)
    if cell == "float":
        assert np.float32(ret).view(np.uint32) == np.float32(want).view(np.uint32)
    else:
        assert ret == want
