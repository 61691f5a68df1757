"""Generated A.4 (fp32 8192^2, pinned host buffers) end to end through the
copy -> kernel -> copy pipeline at several step sizes (codegen.pipe_kb), wall
clock median of 5; one traced run (B2K_PIPE_TRACE=1 prints per-step intervals)."""
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

N = 8192
tp = b2.parse_program(programs.TRANSPOSE_GPU)
a = torch.empty((N, N), dtype=torch.float32, pin_memory=True).numpy()
o = torch.empty((N, N), dtype=torch.float32, pin_memory=True).numpy()
a[...] = np.random.default_rng(0).standard_normal((N, N), dtype=np.float32)
inp = {"in": b2.Array([N, N], a.reshape(-1), "float"), "out": b2.Array([N, N], o.reshape(-1), "float"),
       "W": N, "H": N}
for kb in [0, 8192, 16384, 32768, 65536, 131072]:
    _lib.tune("codegen.pipe_kb", kb)
    b2.run_program(tp, "transpose", inp, backend="codegen")
    ts = []
    for _ in range(5):
        t0 = time.perf_counter()
        b2.run_program(tp, "transpose", inp, backend="codegen")
        ts.append(time.perf_counter() - t0)
    c = codegen.compile_fn(tp.fn("transpose"))
    t = statistics.median(ts)
    print(json.dumps({"pipe_kb": kb, "chunks": c.kernel_piped()[0], "ms": t * 1e3, "GBps": 2 * N * N * 4 / t / 1e9,
                      "ok": bool(np.array_equal(o, a.T))}), flush=True)
t0 = time.perf_counter()
b2.run_program(tp, "transpose", inp, backend="kernels")
t1 = time.perf_counter()
ts = []
for _ in range(5):
    t0 = time.perf_counter()
    b2.run_program(tp, "transpose", inp, backend="kernels")
    ts.append(time.perf_counter() - t0)
print(json.dumps({"hand_written_ms": statistics.median(ts) * 1e3}), flush=True)
