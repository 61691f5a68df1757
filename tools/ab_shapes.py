"""Transpose GB/s over several fp32 / bf16 / fp64 shapes for the library in B2K_LIB."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2605_13864_b200 as b2  # noqa: E402
from paper_2605_13864_b200 import _lib  # noqa: E402


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


out = {"lib": os.path.basename(_lib.LIB_PATH)}
for dt, (R, C) in [(torch.float32, (8192, 16384)), (torch.float32, (16384, 8192)), (torch.float32, (4096, 32768)),
                   (torch.float32, (16384, 16384)), (torch.float32, (32768, 32768)), (torch.bfloat16, (16384, 16384)),
                   (torch.bfloat16, (8192, 16384)), (torch.bfloat16, (4096, 32768)), (torch.bfloat16, (16384, 8192)),
                   (torch.float64, (8192, 8192))]:
    a = torch.empty((R, C), device="cuda", dtype=dt).uniform_()
    o = torch.empty((C, R), device="cuda", dtype=dt)
    ms = timeit(lambda: b2.transpose(a, o))
    out[f"{str(dt)[6:]} {R}x{C}"] = round(2 * a.numel() * a.element_size() / ms / 1e6)
    del a, o
    torch.cuda.empty_cache()
print(json.dumps(out))
