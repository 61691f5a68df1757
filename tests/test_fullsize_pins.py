"""BASELINE C1 (fp32 1024^2 transpose) and C2 (fp32 sum over 2^24) pinned at
FULL size to the reference interpreter itself (tests/golden/fullsize_ref.json,
made by tests/golden/gen_fullsize.py from minigpu.interp.run_program): the CPU
restatements on CPU, the B200 path on the GPU."""
import hashlib
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN
from oracle import oracle, vinterp
from paper_2605_13864_b200 import Array, parse_program, programs


def _pins():
    with open(os.path.join(GOLDEN, "fullsize_ref.json")) as f:
        return json.load(f)


def c1_input(seed):
    return np.random.default_rng(seed).uniform(-1, 1, (1024, 1024)).astype(np.float32)


def c2_input(seed, lo):
    return np.random.default_rng(seed).uniform(lo, 1, 1 << 24).astype(np.float32)


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float32).tobytes()).hexdigest()


def test_c1_restatements_match_reference():
    p = _pins()["C1"]
    a = c1_input(p["seed"])
    assert _sha(oracle.transpose(a)) == p["sha256_out_f32"]
    out = np.zeros(1024 * 1024, np.float32)  # the A.4 GPU-form program through the vectorised restatement
    vinterp.run_program(parse_program(programs.TRANSPOSE_GPU), "transpose",
                        {"in": Array([1024 * 1024], a.reshape(-1), "float"), "out": Array([1024 * 1024], out, "float"),
                         "W": 1024, "H": 1024}, as_numpy=True)
    assert _sha(out) == p["sha256_out_f32"]


def test_c2_restatements_match_reference():
    for p in _pins()["C2"]:
        x = c2_input(p["seed"], p["lo"])
        want = np.uint32(p["result_f32_bits"])
        assert np.float32(oracle.reduce_f32_seq(x)).view(np.uint32) == want
        assert np.float32(oracle.np_reduce_f32_seq(x)).view(np.uint32) == want


@pytest.mark.gpu
def test_c1_gpu_bit_exact():
    import torch

    import paper_2605_13864_b200 as b2
    p = _pins()["C1"]
    a = c1_input(p["seed"])
    assert _sha(b2.transpose(torch.from_numpy(a).cuda()).cpu().numpy()) == p["sha256_out_f32"]
    out = np.zeros(1024 * 1024, np.float32)
    b2.run_program(b2.parse_program(programs.TRANSPOSE_NAIVE), "transpose",
                   {"in": Array([1024, 1024], a.reshape(-1), "float"), "out": Array([1024, 1024], out, "float"),
                    "W": 1024, "H": 1024})
    assert _sha(out) == p["sha256_out_f32"]


@pytest.mark.gpu
def test_c2_gpu_within_tolerance_of_reference():
    import torch

    import paper_2605_13864_b200 as b2
    for p in _pins()["C2"]:
        x = c2_input(p["seed"], p["lo"])
        g = float(b2.reduce_sum(torch.from_numpy(x).cuda()).item())
        exact, absum = oracle.sum_f64(x)
        tol = oracle.f32_tolerance(x.size, exact, absum)
        assert abs(g - exact) <= tol
        # binary64 accumulation: within ~1 ulp of the binary32 result
        assert abs(g - exact) <= oracle.f32_gpu_bound(x.size, exact, absum), (g, exact)
        # against the reference's own pinned value: no further from it than its own
        # measured error plus tol (the old (N-1) u sum|x| bound could not fail)
        assert abs(g - p["result"]) <= oracle.ref_consistency_bound(p["result"], exact, tol)
        ret, _ = b2.run_program(b2.parse_program(programs.source(programs.REDUCE_NAIVE, "float")), "reduce",
                                {"arr": Array([x.size], x, "float"), "N": x.size})
        assert abs(ret - exact) <= tol
