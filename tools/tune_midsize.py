"""Mid-size fp32 transposes (0.5 GB per side): tile walk / tile size sweep."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2605_13864_b200 as b2  # noqa: E402
from paper_2605_13864_b200 import _lib  # noqa: E402


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


for R, C in [(8192, 16384), (16384, 8192), (4096, 32768), (32768, 4096), (16384, 16384)]:
    a = torch.rand((R, C), device="cuda")
    o = torch.empty((C, R), device="cuda")
    nb = 2 * a.numel() * 4
    out = []
    for big, grp in [(1, 0), (1, 16), (1, 8), (1, 1), (0, 0), (0, 4)]:
        _lib.tune("transpose.big", big)
        _lib.tune("transpose.group", grp)
        ms = timeit(lambda: b2.transpose(a, o))
        out.append((big, grp, round(nb / ms / 1e6)))
    _lib.tune("transpose.big", 1)
    _lib.tune("transpose.group", 0)
    print(json.dumps({"shape": [R, C], "results(big,group,GBps)": out}), flush=True)
    del a, o
