"""A/B the transpose between two builds of libb200k on the same box:
python tools/ab_lib.py <path-to-.so>  (prints GB/s for fp32 / fp64 / bf16)."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_13864_b200 import _lib  # noqa: E402

if len(sys.argv) > 1:
    _lib.LIB_PATH = os.path.abspath(sys.argv[1])
import torch  # noqa: E402

import paper_2605_13864_b200 as b2  # noqa: E402


def timeit(fn, reps=20):
    for _ in range(3):
        fn()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)


out = {"lib": _lib.LIB_PATH}
for dtn, (R, C) in [("float32", (32768, 32768)), ("float64", (16384, 32768)), ("bfloat16", (32768, 65536))]:
    dt = getattr(torch, dtn)
    a = torch.empty((R, C), device="cuda", dtype=dt).uniform_()
    o = torch.empty((C, R), device="cuda", dtype=dt)
    ms = timeit(lambda: b2.transpose(a, o))
    out[dtn] = 2 * a.numel() * a.element_size() / ms / 1e6
    del a, o
    torch.cuda.empty_cache()
print(json.dumps(out))
