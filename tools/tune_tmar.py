"""transpose.tma = 2 (TMA-loaded input stages, register transpose, direct stores)
vs the default LDG path, interleaved, plus correctness on ragged shapes."""
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


# correctness first
for R, C in [(512, 256), (1000, 772), (4100, 132), (132, 4100), (4096, 4096)]:
    a = torch.rand((R, C), device="cuda")
    for stages in (2, 3, 4, 6, 7, 8):
        _lib.tune("transpose.tma", 2)
        _lib.tune("transpose.tma_stages", stages)
        o = b2.transpose(a)
        assert torch.equal(o, a.t()), (R, C, stages)
_lib.tune("transpose.tma", 0)
print("correct", flush=True)
res = []
a = torch.rand((32768, 32768), device="cuda")
o = torch.empty_like(a)
nb = 2 * a.numel() * 4
for rep in range(2):
    for tma, stages in [(0, 2), (2, 3), (2, 2), (2, 7), (2, 8)]:
        _lib.tune("transpose.tma", tma)
        _lib.tune("transpose.tma_stages", stages)
        ms = timeit(lambda: b2.transpose(a, o))
        res.append({"tma": tma, "stages": stages, "GBps": nb / ms / 1e6, "ok": bool(torch.equal(o, a.t()))})
        print(json.dumps(res[-1]), flush=True)
_lib.tune("transpose.tma", 0)
_lib.tune("transpose.tma_stages", 2)
os.makedirs("gpurun_out", exist_ok=True)
json.dump(res, open("gpurun_out/tune_tmar.json", "w"), indent=1)
