"""Column-major tile walk (transpose.group >= tiles_r) across tile shapes and
residencies: concurrent CTAs then work down one column block, so their output
rows are written as long contiguous runs (the group sweep showed the write side
dominates DRAM efficiency)."""
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
FULL = 1 << 20
plans = {
    "float32": ((32768, 32768), [(7, [1]), (9, [1]), (10, [1]), (5, [1, 2, 3]), (8, [1, 2, 3]),
                                 (1, [2, 4, 6]), (2, [2, 4, 6]), (0, [4, 8])]),
    "float64": ((16384, 32768), [(7, [1]), (2, [1, 2, 3]), (0, [2, 4])]),
    "bfloat16": ((32768, 65536), [(0, [1, 2, 3]), (1, [2, 4]), (2, [2, 4]), (7, [1])]),
}
for dtn, ((R, C), plan) in plans.items():
    dt = getattr(torch, dtn)
    a = torch.empty((R, C), device="cuda", dtype=dt).uniform_()
    o = torch.empty((C, R), device="cuda", dtype=dt)
    nb = 2 * a.numel() * a.element_size()
    _lib.tune("transpose.big", 0)
    for var, cpss in plan:
        for cps in cpss:
            for grp in [FULL, 64, 16, 1]:
                _lib.tune("transpose.variant", var)
                _lib.tune("transpose.ctas_per_sm", cps)
                _lib.tune("transpose.group", grp)
                try:
                    med, best = timeit(lambda: b2.transpose(a, o))
                except Exception as e:  # noqa: BLE001
                    print("fail", var, cps, grp, e)
                    continue
                ok = bool(torch.equal(o, a.t()))
                res.append({"dtype": dtn, "variant": var, "cps": cps, "group": grp, "ms": med,
                            "GBps": nb / med / 1e6, "best_GBps": nb / best / 1e6, "ok": ok})
                print(json.dumps(res[-1]), flush=True)
    for k in ("transpose.variant", "transpose.ctas_per_sm", "transpose.group"):
        _lib.tune(k, 0)
    _lib.tune("transpose.big", 1)
    del a, o
    torch.cuda.empty_cache()
os.makedirs("gpurun_out", exist_ok=True)
json.dump(res, open("gpurun_out/tune_colwalk.json", "w"), indent=1)
