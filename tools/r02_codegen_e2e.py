"""End-to-end run_program of the generated A.4 / A.5 programs (backend="codegen")
with and without the chunked copy -> kernel -> copy pipeline, against the
hand-written host pipeline (backend="kernels" -> b2_transpose_host /
b2_reduce_tree512_host) on the same host buffers; pinned and pageable. Wall clock
of the whole call (copies included), median of 5 after one warm-up."""
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2605_13864_b200 as b2  # noqa: E402
from paper_2605_13864_b200 import _lib, codegen, programs  # noqa: E402


def wall(fn, reps=5):
    fn()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return statistics.median(ts)


def bufs(shape, pinned):
    if pinned:
        return torch.empty(shape, dtype=torch.float32, pin_memory=True).numpy()
    return np.empty(shape, np.float32)


N = int(os.environ.get("E2E_N", "8192"))
tp = b2.parse_program(programs.TRANSPOSE_GPU)
rp = b2.parse_program(programs.REDUCE_TREE_F32)
res = []
for pinned in (True, False):
    a, o = bufs((N, N), pinned), bufs((N, N), pinned)
    a[...] = np.random.default_rng(0).standard_normal((N, N), dtype=np.float32)
    inp = {"in": b2.Array([N, N], a.reshape(-1), "float"), "out": b2.Array([N, N], o.reshape(-1), "float"),
           "W": N, "H": N}
    nbytes = 2 * N * N * 4
    rec = {"program": f"A.4 transpose fp32 {N}x{N}", "pinned": pinned, "bytes_moved": nbytes}
    for label, backend, kb in [("hand_written", "kernels", None), ("codegen_pipelined", "codegen", 65536),
                               ("codegen_program_order", "codegen", 0)]:
        if kb is not None:
            _lib.tune("codegen.pipe_kb", kb)
        o[...] = 0
        t = wall(lambda: b2.run_program(tp, "transpose", inp, backend=backend))
        ok = bool(np.array_equal(o, a.T))
        rec[label] = {"ms": t * 1e3, "GBps": nbytes / t / 1e9, "ok": ok}
        if backend == "codegen":
            c = codegen.compile_fn(tp.fn("transpose"))
            rec[label]["chunks"] = c.kernel_piped()[0]
            rec[label]["kernel_ms"] = c.kernel_ms()[0]
    _lib.tune("codegen.pipe_kb", 65536)
    print(json.dumps(rec), flush=True)
    res.append(rec)
    del a, o, inp

M = int(os.environ.get("E2E_M", str(1 << 26)))
for pinned in (True, False):
    x = bufs((M,), pinned)
    x[...] = np.random.default_rng(1).uniform(-1, 1, M).astype(np.float32)
    inp = {"arr": b2.Array([M], x, "float"), "N": M}
    rec = {"program": f"A.5 tree reduce fp32 n={M}", "pinned": pinned, "bytes_moved": M * 4}
    want = None
    for label, backend, kb in [("hand_written", "kernels", None), ("codegen_pipelined", "codegen", 65536),
                               ("codegen_program_order", "codegen", 0)]:
        if kb is not None:
            _lib.tune("codegen.pipe_kb", kb)
        out = []
        t = wall(lambda: out.append(b2.run_program(rp, "reduce", inp, backend=backend)[0]))
        want = out[-1] if want is None else want
        rec[label] = {"ms": t * 1e3, "GBps": M * 4 / t / 1e9, "same_bits_as_hand_written": out[-1] == want}
        if backend == "codegen":
            c = codegen.compile_fn(rp.fn("reduce"))
            rec[label]["chunks"] = c.kernel_piped()[0]
    _lib.tune("codegen.pipe_kb", 65536)
    print(json.dumps(rec), flush=True)
