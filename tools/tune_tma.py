"""TMA transpose vs LDG transpose on B200 (fp32 32768^2 and odd shapes)."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2605_13864_b200 as b2  # noqa: E402
from paper_2605_13864_b200 import _lib  # noqa: E402

res = []


def timeit(fn, reps=10):
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


dev = torch.device("cuda", 0)
for (R, C) in [(32768, 32768), (16384, 65536), (32000, 32008)]:
    a = torch.empty((R, C), device=dev).uniform_()
    o = torch.empty((C, R), device=dev)
    nb = 2 * a.numel() * 4
    _lib.tune("transpose.tma", 0)
    ms = timeit(lambda: b2.transpose(a, o))
    res.append({"shape": [R, C], "path": "ldg", "ms": ms, "GBps": nb / ms / 1e6})
    print(json.dumps(res[-1]), flush=True)
    for stages in [2, 3, 4, 6]:
        for cps in [1, 2]:
            if (stages + 2) * 16 * cps > 220:
                continue
            for grp in [1, 4]:
                _lib.tune("transpose.tma", 1)
                _lib.tune("transpose.tma_stages", stages)
                _lib.tune("transpose.ctas_per_sm", cps)
                _lib.tune("transpose.group", grp)
                o.zero_()
                ms = timeit(lambda: b2.transpose(a, o))
                ok = bool(torch.equal(o, a.t()))
                res.append({"shape": [R, C], "path": "tma", "stages": stages, "cps": cps, "group": grp,
                            "ms": ms, "GBps": nb / ms / 1e6, "ok": ok})
                print(json.dumps(res[-1]), flush=True)
    _lib.tune("transpose.tma", 0)
    _lib.tune("transpose.ctas_per_sm", 0)
    _lib.tune("transpose.group", 4)
    del a, o
    torch.cuda.empty_cache()
os.makedirs("gpurun_out", exist_ok=True)
json.dump(res, open("gpurun_out/tune_tma.json", "w"), indent=1)
