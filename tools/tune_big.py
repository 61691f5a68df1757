"""Large-tile transpose variants (fewer, longer DRAM streams) vs the tuned default."""
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


SWEEP = {
    "float32": ((32768, 32768), [(0, [0]), (7, [1]), (8, [1, 2]), (9, [1]), (10, [1])]),
    "bfloat16": ((32768, 65536), [(0, [0]), (7, [1])]),
    "float64": ((16384, 32768), [(0, [0]), (7, [1])]),
}
for dtn, ((R, C), plan) in SWEEP.items():
    dt = getattr(torch, dtn)
    a = torch.empty((R, C), device="cuda", dtype=dt).uniform_()
    o = torch.empty((C, R), device="cuda", dtype=dt)
    nb = 2 * a.numel() * a.element_size()
    for var, cpss in plan:
        for cps in cpss:
            for grp in [1, 2, 4]:
                _lib.tune("transpose.variant", var)
                _lib.tune("transpose.ctas_per_sm", cps)
                _lib.tune("transpose.group", grp)
                o.zero_()
                ms = timeit(lambda: b2.transpose(a, o))
                ok = bool(torch.equal(o, a.t()))
                res.append({"dtype": dtn, "variant": var, "cps": cps, "group": grp, "ms": ms,
                            "GBps": nb / ms / 1e6, "ok": ok})
                print(json.dumps(res[-1]), flush=True)
    del a, o
    torch.cuda.empty_cache()
os.makedirs("gpurun_out", exist_ok=True)
json.dump(res, open("gpurun_out/tune_big.json", "w"), indent=1)
