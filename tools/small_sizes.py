"""Latency-bound sizes (BASELINE C1 1024^2 transpose, C2 2^24 fp32 sum, the
paper's 4096^2): cold-L2 (read-pass flush) CUDA-event times per launch, default
knobs vs reduce variants / residencies."""
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
res = []


def timeit(fn, reps=25):
    ts = []
    for i in range(reps + 3):
        flush.sum()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        if i >= 3:
            ts.append(e0.elapsed_time(e1))
    return statistics.median(ts) * 1e3, min(ts) * 1e3


def rec(**kw):
    res.append(kw)
    print(json.dumps(kw), flush=True)


empty = torch.empty(0, device="cuda")
us, best = timeit(lambda: torch.cuda._sleep(0))
rec(what="empty event pair", us=us)
for logn in [20, 22, 24, 26]:
    x = torch.rand(1 << logn, device="cuda")
    r = torch.empty(1, device="cuda")
    for var in range(5):
        for cps in [0, 2, 4]:
            _lib.tune("reduce.variant", var)
            _lib.tune("reduce.ctas_per_sm", cps)
            us, best = timeit(lambda: b2.reduce_sum(x, out=r))
            rec(what="reduce f32", log2n=logn, variant=var, cps=cps, us=us, best_us=best,
                GBps=x.numel() * 4 / us / 1e3)
    _lib.tune("reduce.variant", 0)
    _lib.tune("reduce.ctas_per_sm", 0)
for n in [1024, 2048, 4096]:
    a = torch.rand((n, n), device="cuda")
    o = torch.empty_like(a)
    for var, cps in [(0, 0), (0, 2), (0, 8), (5, 0), (7, 0)]:
        _lib.tune("transpose.variant", var)
        _lib.tune("transpose.ctas_per_sm", cps)
        _lib.tune("transpose.big", 0)
        us, best = timeit(lambda: b2.transpose(a, o))
        rec(what="transpose f32", n=n, variant=var, cps=cps, us=us, best_us=best, GBps=2 * n * n * 4 / us / 1e3)
    _lib.tune("transpose.variant", 0)
    _lib.tune("transpose.ctas_per_sm", 0)
    _lib.tune("transpose.big", 1)
os.makedirs("gpurun_out", exist_ok=True)
json.dump(res, open("gpurun_out/small_sizes.json", "w"), indent=1)
