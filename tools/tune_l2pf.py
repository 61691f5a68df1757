"""L2 bulk-prefetch distance for the vector transpose (transpose.l2_prefetch)."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2605_13864_b200 as b2  # noqa: E402
from paper_2605_13864_b200 import _lib  # noqa: E402


def timeit(fn, reps=15):
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


res = []
for dtn, (R, C) in [("float32", (32768, 32768)), ("bfloat16", (32768, 65536)), ("float64", (16384, 32768))]:
    dt = getattr(torch, dtn)
    a = torch.empty((R, C), device="cuda", dtype=dt).uniform_()
    o = torch.empty((C, R), device="cuda", dtype=dt)
    nb = 2 * a.numel() * a.element_size()
    for rep in range(2):
        for pf in [0, 1, 2, 3]:
            _lib.tune("transpose.l2_prefetch", pf)
            ms = timeit(lambda: b2.transpose(a, o))
            res.append({"dtype": dtn, "pf": pf, "rep": rep, "GBps": nb / ms / 1e6, "ok": bool(torch.equal(o, a.t()))})
            print(json.dumps(res[-1]), flush=True)
    _lib.tune("transpose.l2_prefetch", 0)
    del a, o
    torch.cuda.empty_cache()
os.makedirs("gpurun_out", exist_ok=True)
json.dump(res, open("gpurun_out/tune_l2pf.json", "w"), indent=1)
