"""The A.4 / A.5 derivation families on the HAND-WRITTEN kernels (recognised by
parameter, recognize.family_candidates): every tile-size member transposes
bit-exactly; every block-size member of the tree reduction reproduces the
reference interpreter's association bit for bit (tree_kernel<B>), checked
against the family's numpy restatement (pinned to the reference in
tests/golden/families_pinned.json) and against the generated kernels."""
import numpy as np
import pytest
import torch

import paper_2605_13864_b200 as b2
from program_families import np_reduce_family, reduce_family, transpose_family

pytestmark = pytest.mark.gpu


def _np_tree_partials(x, B):
    b = x.reshape(-1, B)
    s = b[:, 0::2] + b[:, 1::2]
    h = B // 4
    while h >= 1:
        s = s.copy()
        s[:, :h] = s[:, :h] + s[:, h:2 * h]
        h //= 2
    return s[:, 0].copy()


@pytest.mark.parametrize("B", [64, 128, 256, 512, 1024, 2048])
def test_tree_kernel_partials_bit_exact(B):
    rng = np.random.default_rng(B)
    x = rng.standard_normal(B * 1531).astype(np.float32)
    t = torch.from_numpy(x).cuda()
    got = b2.reduce_tree_partials(t, B).cpu().numpy()
    assert np.array_equal(got.view(np.uint32), _np_tree_partials(x, B).view(np.uint32))
    want = np_reduce_family(x, B)
    assert np.float32(b2.reduce_tree(t, B)).view(np.uint32) == np.float32(want).view(np.uint32)
    assert np.float32(b2.reduce_tree(x, B)).view(np.uint32) == np.float32(want).view(np.uint32)


@pytest.mark.parametrize("B,cell", [(64, "float"), (128, "int"), (256, "float"), (1024, "float"),
                                    (2048, "int"), (512, "int"), (2048, "float")])
def test_reduce_family_on_hand_written_kernels(B, cell):
    rng = np.random.default_rng(B + 7)
    n = B * 300
    x = rng.uniform(-1, 1, n).astype(np.float32) if cell == "float" else \
        rng.integers(-2**31, 2**31, n, dtype=np.int64).astype(np.int32)
    p = b2.parse_program(reduce_family(B, cell))
    n0 = b2.launch_count()
    got, _ = b2.run_program(p, "reduce", {"arr": b2.Array([n], x, cell), "N": n}, backend="kernels")
    assert b2.launch_count() > n0
    want = np_reduce_family(x, B)
    if cell == "float":
        assert np.float32(got).view(np.uint32) == np.float32(want).view(np.uint32)
        gen, _ = b2.run_program(p, "reduce", {"arr": b2.Array([n], x, cell), "N": n}, backend="codegen")
        assert np.float32(gen).view(np.uint32) == np.float32(got).view(np.uint32)
    else:
        assert got == want


@pytest.mark.parametrize("T,R", [(8, 2), (16, 16), (32, 4), (64, 8), (64, 16), (128, 8)])
def test_transpose_family_on_hand_written_kernels(T, R):
    rng = np.random.default_rng(T * R)
    H, W = 7 * T, 5 * T
    a = rng.standard_normal((H, W)).astype(np.float32)
    out = np.zeros(H * W, np.float32)
    b2.run_program(b2.parse_program(transpose_family(T, R)), "transpose",
                   {"in": b2.Array([H * W], a.reshape(-1), "float"), "out": b2.Array([H * W], out, "float"),
                    "W": W, "H": H}, backend="kernels")
    assert np.array_equal(out.reshape(W, H), a.T)


def test_family_exact_div_errors():
    with pytest.raises(b2.InterpError, match=r"exact_div\(100, 64\) is not exact"):
        b2.run_program(b2.parse_program(transpose_family(64, 8)), "transpose",
                       {"in": [0.0] * 6400, "out": [0.0] * 6400, "W": 100, "H": 64})
    with pytest.raises(b2.InterpError, match=r"exact_div\(300, 256\) is not exact"):
        b2.run_program(b2.parse_program(reduce_family(256, "float")), "reduce", {"arr": [1.0] * 300, "N": 300})
