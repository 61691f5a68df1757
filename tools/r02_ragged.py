"""TMA-staged (transpose.tma = 1) vs LDG-staged (default) fp32 transposes on
ragged, 16-B-aligned shapes (cols not a multiple of the 128-column tile), A B A B
interleaved on one box; CUDA-event median of 10 launches (inputs > L2)."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2605_13864_b200 as b2  # noqa: E402
from paper_2605_13864_b200 import _lib  # noqa: E402


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


shapes = [(32768, 32768), (32000, 32008), (30000, 30004), (32768, 32764), (32764, 32768), (20000, 40004),
          (12288, 50004), (8000, 8004), (4096, 4100), (16384, 16388)]
for (R, C) in shapes:
    a = torch.empty((R, C), device="cuda").uniform_()
    o = torch.empty((C, R), device="cuda")
    nb = 2 * a.numel() * 4
    rec = {"shape": [R, C]}
    for rep in range(2):
        for tma in (0, 1):
            _lib.tune("transpose.tma", tma)
            ms = timeit(lambda: b2.transpose(a, o))
            rec.setdefault(f"tma{tma}", []).append(round(nb / ms / 1e6, 1))
    _lib.tune("transpose.tma", 0)
    o.zero_()
    _lib.tune("transpose.tma", 1)
    b2.transpose(a, o)
    rec["tma_ok"] = bool(torch.equal(o, a.t()))
    _lib.tune("transpose.tma", 0)
    print(json.dumps(rec), flush=True)
    del a, o
    torch.cuda.empty_cache()
