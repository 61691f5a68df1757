"""Reduce variants incl. 256-bit loads (reduce.variant 5-8: LDG.E.256) on C3-sized
inputs, interleaved repeats."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_13864_b200 import _lib  # noqa: E402

if len(sys.argv) > 1:
    _lib.LIB_PATH = os.path.abspath(sys.argv[1])
import torch  # noqa: E402

import paper_2605_13864_b200 as b2  # noqa: E402


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


res = []
n = 1 << 30
xi = torch.randint(-2**31, 2**31, (n,), device="cuda", dtype=torch.int64).to(torch.int32)
xf = torch.rand(n, device="cuda")
oi = torch.empty(1, dtype=torch.int64, device="cuda")
of = torch.empty(1, device="cuda")
want = int(xi.to(torch.int64).sum())
for rep in range(2):
    for v in [0, 5, 6, 7, 8, 1]:
        _lib.tune("reduce.variant", v)
        for name, x, o in [("int32", xi, oi), ("float32", xf, of)]:
            ms = timeit(lambda: b2.reduce_sum(x, out=o))
            ok = (int(o.item()) == want) if name == "int32" else True
            res.append({"lib": _lib.LIB_PATH, "variant": v, "dtype": name, "GBps": (4 * n + 8) / ms / 1e6, "ok": ok})
            print(json.dumps(res[-1]), flush=True)
_lib.tune("reduce.variant", 0)
os.makedirs("gpurun_out", exist_ok=True)
with open("gpurun_out/tune_reduce_wide.json", "a") as f:
    f.write(json.dumps(res) + "\n")
