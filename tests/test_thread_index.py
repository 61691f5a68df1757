"""SPEC acceptance 9 (thread-index oracle): for random `thread for` nests
(<= 4 loops, concrete bounds, grid <= 4096) the index expressions evaluated at
every thread reproduce the row-major nest coordinates — through the generated
kernels on the GPU, the vectorised interpreter restatement and the gate (which
must see no race: every thread writes its own cell)."""
import numpy as np
import pytest

from oracle import vinterp
from paper_2605_13864_b200 import check_kernels, parse_program
from program_families import np_thread_index, thread_index_nests, thread_index_program

NESTS = thread_index_nests(100, seed=9)
TOTAL = int(sum(np.prod(b) for b, _ in NESTS))


def test_nests_are_valid():
    for bounds, tpb in NESTS:
        assert 1 <= len(bounds) <= 4 and np.prod(bounds) <= 4096 and np.prod(bounds) % tpb == 0 and tpb <= 1024


def test_vinterp_and_gate_on_nests():
    prog = parse_program(thread_index_program(NESTS))
    rep = check_kernels(prog, "idx", {"res": [0] * TOTAL, "N": TOTAL})
    assert rep["kernels"] == len(NESTS)
    _, outs = vinterp.run_program(prog, "idx", {"res": [0] * TOTAL, "N": TOTAL})
    assert np.array_equal(np.array(outs["res"], dtype=np.int64), np_thread_index(NESTS))


@pytest.mark.gpu
def test_generated_kernels_on_nests():
    import paper_2605_13864_b200 as b2
    res = np.zeros(TOTAL, np.int32)
    b2.run_program(parse_program(thread_index_program(NESTS)), "idx", {"res": b2.Array([TOTAL], res, "int"),
                                                                       "N": TOTAL}, backend="codegen")
    assert np.array_equal(res.astype(np.int64), np_thread_index(NESTS))


def test_reference_interpreter_agrees():
    from conftest import reference_available
    if not reference_available():
        pytest.skip("reference only in the build container")
    from minigpu.interp import run_program as rrun
    from minigpu.parser import parse_program as rparse
    _, outs = rrun(rparse(thread_index_program(NESTS[:30])), "idx",
                   {"res": [0] * int(sum(np.prod(b) for b, _ in NESTS[:30])), "N": int(sum(np.prod(b) for b, _ in NESTS[:30]))})
    assert np.array_equal(np.array(outs["res"], dtype=np.int64), np_thread_index(NESTS[:30]))


def test_chunk_partition_property():
    """SPEC.md:530 (acceptance 7): for all (n, M) with n | M, M <= 64, the n chunks a
    `thread for` of n iterations gives a context of M threads (interp.py:285-289:
    width M / n each; the decomposition the code generator emits, rel / (M/n) and
    rel % (M/n)) partition 0..M exactly: contiguous, disjoint, covering."""
    for M in range(1, 65):
        for n in range(1, M + 1):
            if M % n:
                continue
            w = M // n
            owner = [rel // w for rel in range(M)]
            pos = [rel % w for rel in range(M)]
            for i in range(n):
                chunk = [rel for rel in range(M) if owner[rel] == i]
                assert chunk == list(range(i * w, (i + 1) * w))
                assert [pos[r] for r in chunk] == list(range(w))
