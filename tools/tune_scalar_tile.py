"""Odd-pitch 2-byte transposes: padded scalar tile 64 vs 128 (transpose.scalar_tile),
residency (transpose.scalar_ctas), interleaved."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2605_13864_b200 as b2  # noqa: E402
from paper_2605_13864_b200 import _lib  # noqa: E402

L2 = 126 * 1024 * 1024
flush = torch.ones(2 * L2 // 4, device="cuda")


def timeit(fn, nb, reps=15):
    cold = nb < 4 * L2
    for _ in range(3):
        fn()
    ts = []
    for _ in range(reps):
        if cold:
            flush.sum()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)


res = []
for R, C in [(4097, 8191), (16385, 16383)]:
    a = torch.empty((R, C), device="cuda", dtype=torch.bfloat16).uniform_()
    o = torch.empty((C, R), device="cuda", dtype=torch.bfloat16)
    nb = 2 * a.numel() * 2
    for rep in range(2):
        for ts_, cps in [(0, 0), (0, 4), (128, 0), (128, 2), (128, 3)]:
            _lib.tune("transpose.scalar_tile", ts_)
            _lib.tune("transpose.scalar_ctas", cps)
            ms = timeit(lambda: b2.transpose(a, o), nb)
            ok = bool(torch.equal(o, a.t()))
            res.append({"shape": [R, C], "tile": ts_ or 64, "cps": cps, "GBps": nb / ms / 1e6, "ok": ok})
            print(json.dumps(res[-1]), flush=True)
    _lib.tune("transpose.scalar_tile", 0)
    _lib.tune("transpose.scalar_ctas", 0)
    del a, o
os.makedirs("gpurun_out", exist_ok=True)
json.dump(res, open("gpurun_out/tune_scalar_tile.json", "w"), indent=1)
