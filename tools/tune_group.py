"""Band height (transpose.group) sweep for the 128-KB fp32/fp64 tiles: the
concurrent window of ~#SM tiles covers `group` tile-rows x #SM/group tile-columns,
trading aggregate read-stream length (long rows) for write-stream length."""
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
    return statistics.median(ts), min(ts)


res = []
for dtn, (R, C) in [("float32", (32768, 32768)), ("float64", (16384, 32768))]:
    dt = getattr(torch, dtn)
    a = torch.empty((R, C), device="cuda", dtype=dt).uniform_()
    o = torch.empty((C, R), device="cuda", dtype=dt)
    nb = 2 * a.numel() * a.element_size()
    for grp in [1, 2, 3, 4, 6, 8, 12, 16, 24, 32, 48, 64, 128]:
        _lib.tune("transpose.group", grp)
        med, best = timeit(lambda: b2.transpose(a, o))
        res.append({"dtype": dtn, "group": grp, "ms": med, "GBps": nb / med / 1e6, "best_GBps": nb / best / 1e6})
        print(json.dumps(res[-1]), flush=True)
    _lib.tune("transpose.group", 0)
    assert torch.equal(o, a.t())
    del a, o
    torch.cuda.empty_cache()
os.makedirs("gpurun_out", exist_ok=True)
json.dump(res, open("gpurun_out/tune_group.json", "w"), indent=1)
