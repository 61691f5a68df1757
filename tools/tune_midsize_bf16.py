"""Mid-size bf16 / fp64 transposes (0.25-1 GB per side): tile shape x walk x
residency sweep (CUDA-event medians; inputs larger than L2)."""
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


# (variant, group, ctas_per_sm); group -1 = column walk (group = tiles_r)
SETS = {
    torch.bfloat16: [(0, 0, 0), (0, 1, 0), (0, 2, 0), (0, 8, 0), (0, 0, 1), (0, 1, 1), (0, 0, 3),
                     (7, 0, 0), (7, 1, 0), (7, 4, 0), (1, 0, 0), (1, 1, 0), (2, 0, 0)],
    torch.float64: [(0, 0, 0), (0, 1, 0), (0, 2, 0), (0, 8, 0), (0, 0, 1), (0, 0, 3), (2, 0, 0), (2, 1, 0),
                    (7, 0, 0), (7, 1, 0)],
}
for dt, shapes in [(torch.bfloat16, [(8192, 16384), (16384, 8192), (4096, 32768), (16384, 16384),
                                     (32768, 65536)]),
                   (torch.float64, [(8192, 8192), (4096, 16384), (16384, 4096), (16384, 16384)])]:
    for R, C in shapes:
        a = torch.empty((R, C), device="cuda", dtype=dt).uniform_()
        o = torch.empty((C, R), device="cuda", dtype=dt)
        nb = 2 * a.numel() * a.element_size()
        res = []
        for var, grp, cps in SETS[dt]:
            _lib.tune("transpose.variant", var)
            _lib.tune("transpose.group", grp)
            _lib.tune("transpose.ctas_per_sm", cps)
            ms = timeit(lambda: b2.transpose(a, o))
            res.append(((var, grp, cps), round(nb / ms / 1e6)))
        for k in ("transpose.variant", "transpose.group", "transpose.ctas_per_sm"):
            _lib.tune(k, 0)
        assert torch.equal(o, a.t())
        print(json.dumps({"dtype": str(dt), "shape": [R, C], "results((var,group,cps),GBps)": res}), flush=True)
        del a, o
        torch.cuda.empty_cache()
