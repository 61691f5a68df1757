"""TMA-staged transpose with the column-major tile walk: stages x CTAs/SM x walk."""
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
R = C = 32768
a = torch.empty((R, C), device="cuda").uniform_()
o = torch.empty((C, R), device="cuda")
nb = 2 * a.numel() * 4
ms = timeit(lambda: b2.transpose(a, o))
res.append({"path": "default LDG", "GBps": nb / ms / 1e6})
print(json.dumps(res[-1]), flush=True)
_lib.tune("transpose.tma", 1)
for grp in [1 << 20, 1]:
    for stages in [2, 3, 4, 6]:
        for cps in [1, 2, 3, 4]:
            _lib.tune("transpose.group", grp)
            _lib.tune("transpose.tma_stages", stages)
            _lib.tune("transpose.ctas_per_sm", cps)
            try:
                ms = timeit(lambda: b2.transpose(a, o))
            except Exception as e:  # noqa: BLE001
                print("fail", grp, stages, cps, e)
                continue
            ok = bool(torch.equal(o, a.t()))
            res.append({"path": "tma", "group": grp, "stages": stages, "cps": cps, "GBps": nb / ms / 1e6, "ok": ok})
            print(json.dumps(res[-1]), flush=True)
os.makedirs("gpurun_out", exist_ok=True)
json.dump(res, open("gpurun_out/tune_tma_colwalk.json", "w"), indent=1)
