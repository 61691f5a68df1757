"""The naive fp32 program A.2 in the reference's own order (b2_reduce_sum_seq_f32,
run_program(..., fp_order="reference")): bit-identical with the reference interpreter
— at BASELINE C2's full 2^24 cells against the reference's pinned result bits
(tests/golden/fullsize_ref.json, produced by minigpu.interp itself), on the golden
cases, across host-pipeline chunks and chained device calls."""
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _seq_f32(x: np.ndarray) -> np.float32:
    """Restatement of the reference's loop (interp.py:262-270): binary32 rounding
    after every add; numpy cumsum in float32 is the same left fold."""
    return np.cumsum(x, dtype=np.float32)[-1] if x.size else np.float32(0)


def _pins():
    with open(os.path.join(GOLDEN, "fullsize_ref.json")) as f:
        return json.load(f)["C2"]


def test_c2_full_size_bit_identical_to_the_reference():
    import paper_2605_13864_b200 as b2
    from paper_2605_13864_b200 import programs
    for p in _pins():
        x = np.random.default_rng(p["seed"]).uniform(p["lo"], 1, p["n"]).astype(np.float32)
        want = np.uint32(p["result_f32_bits"])
        assert np.float32(b2.reduce_sum_sequential(x)).view(np.uint32) == want, p["seed"]  # host pipeline
        dev = b2.reduce_sum_sequential(torch.from_numpy(x).cuda())                       # device entry
        assert np.float32(dev.item()).view(np.uint32) == want, p["seed"]
        ret, _ = b2.run_program(b2.parse_program(programs.source(programs.REDUCE_NAIVE, "float")), "reduce",
                                {"arr": b2.Array([x.size], x, "float"), "N": x.size}, fp_order="reference")
        assert np.float32(ret).view(np.uint32) == want, p["seed"]


def test_golden_naive_fp32_sums_bit_identical(golden):
    import paper_2605_13864_b200 as b2
    from paper_2605_13864_b200 import programs
    prog = b2.parse_program(programs.source(programs.REDUCE_NAIVE, "float"))
    seen = 0
    for c in golden:
        if c["kind"] != "reduce" or "result_int" in c or "tree" in c["program"]:
            continue
        x = c["inp"]
        ret, _ = b2.run_program(prog, "reduce", {"arr": x.tolist(), "N": int(x.size)}, fp_order="reference")
        assert np.float32(ret).view(np.uint32) == np.uint32(c["result_f32_bits"]), c["id"]
        seen += 1
    assert seen > 0


@pytest.mark.parametrize("n", [0, 1, 2, 5, 2047, 2048, 2049, 4096 * 3 + 7, 1 << 18])
@pytest.mark.parametrize("off", [0, 1, 3])
def test_ragged_and_misaligned(n, off):
    import paper_2605_13864_b200 as b2
    rng = np.random.default_rng(n * 7 + off)
    h = (rng.standard_normal(n + off) * np.exp2(rng.integers(-30, 30, n + off))).astype(np.float32)
    x = h[off:]
    want = _seq_f32(x).view(np.uint32)
    got = b2.reduce_sum_sequential(torch.from_numpy(h).cuda()[off:])
    assert np.float32(got.item()).view(np.uint32) == want
    assert np.float32(b2.reduce_sum_sequential(x)).view(np.uint32) == want


def test_host_chunks_and_chained_device_calls():
    """1-MiB host-pipeline chunks are summed in order; two device calls chain through
    the accumulator exactly like one call over the concatenation."""
    import paper_2605_13864_b200 as b2
    from paper_2605_13864_b200 import _lib
    rng = np.random.default_rng(11)
    x = rng.uniform(-1, 1, 3 * (1 << 18) + 5).astype(np.float32)
    want = _seq_f32(x).view(np.uint32)
    prev = _lib.tuning("host.chunk_mb")
    _lib.tune("host.chunk_mb", 1)
    try:
        assert np.float32(b2.reduce_sum_sequential(x)).view(np.uint32) == want
    finally:
        _lib.tune("host.chunk_mb", prev)
    d = torch.from_numpy(x).cuda()
    acc = torch.zeros(1, dtype=torch.float32, device="cuda")
    L = _lib.lib()
    k = 300_001
    for a, b in ((0, k), (k, x.size)):
        _lib.check(L.b2_reduce_sum_seq_f32(d[a:].data_ptr(), b - a, acc.data_ptr(), 0,
                                           torch.cuda.current_stream().cuda_stream))
    assert np.float32(acc.item()).view(np.uint32) == want
