"""Finer sweep: transpose {variant x ctas_per_sm x group} per dtype; reduce
{variant x ctas_per_sm}. CUDA-event median of REPS launches; inputs >> L2."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2605_13864_b200 as b2  # noqa: E402
from paper_2605_13864_b200 import _lib  # noqa: E402

results = []


def timeit(fn, reps=10, warm=2):
    for _ in range(warm):
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


def rec(**kw):
    results.append(kw)
    print(json.dumps(kw), flush=True)


dev = torch.device("cuda", 0)
xi = torch.randint(-2**31, 2**31, (1 << 30,), device=dev, dtype=torch.int64).to(torch.int32)
r = torch.empty(1, dtype=torch.int64, device=dev)
for var, cpss in [(0, [1, 2, 3, 4]), (3, [1, 2]), (2, [2, 3, 4, 5, 6, 8]), (1, [1, 2, 3, 4])]:
    for cps in cpss:
        _lib.tune("reduce.variant", var)
        _lib.tune("reduce.ctas_per_sm", cps)
        ms = timeit(lambda: b2.reduce_sum(xi, out=r))
        rec(what="reduce_i32", variant=var, cps=cps, ms=ms, GBps=xi.numel() * 4 / ms / 1e6)
_lib.tune("reduce.variant", 0)
_lib.tune("reduce.ctas_per_sm", 0)
del xi
torch.cuda.empty_cache()

sweep = {"float32": (32768, 32768, [0, 1, 2, 3, 4]), "bfloat16": (32768, 65536, [0, 1, 2]),
         "float64": (16384, 32768, [0, 1, 2])}
for dtn, (R, C, variants) in sweep.items():
    dt = getattr(torch, dtn)
    a = torch.empty((R, C), device=dev, dtype=dt).uniform_()
    o = torch.empty((C, R), device=dev, dtype=dt)
    nbytes = 2 * a.numel() * a.element_size()
    for var in variants:
        for cps in [1, 2, 3, 4, 5, 6]:
            for grp in [1, 4, 16]:
                _lib.tune("transpose.variant", var)
                _lib.tune("transpose.ctas_per_sm", cps)
                _lib.tune("transpose.group", grp)
                ms = timeit(lambda: b2.transpose(a, o))
                rec(what=f"transpose_{dtn}", variant=var, cps=cps, group=grp, ms=ms, GBps=nbytes / ms / 1e6)
        torch.cuda.synchronize()
        assert torch.equal(o[-256:, -256:], a[-256:, -256:].t())
    del a, o
    torch.cuda.empty_cache()
os.makedirs("gpurun_out", exist_ok=True)
with open("gpurun_out/tune2.json", "w") as f:
    json.dump(results, f, indent=1)
