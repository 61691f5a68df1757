"""Large odd-pitch transposes: scalar-tile residency per element size."""
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
for dt, (R, C) in [(torch.float32, (16385, 16383)), (torch.float64, (8193, 16383)), (torch.float32, (4097, 8191)),
                   (torch.float64, (4097, 8191)), (torch.bfloat16, (16385, 32767))]:
    a = torch.empty((R, C), device="cuda", dtype=dt).uniform_()
    o = torch.empty((C, R), device="cuda", dtype=dt)
    nb = 2 * a.numel() * a.element_size()
    for cps in [0, 1, 2, 3, 4, 6]:
        for tile in ([0, 128] if dt == torch.bfloat16 else [0]):
            _lib.tune("transpose.scalar_ctas", cps)
            _lib.tune("transpose.scalar_tile", tile)
            ms = timeit(lambda: b2.transpose(a, o))
            res.append({"dtype": str(dt), "shape": [R, C], "cps": cps, "tile": tile or 64, "GBps": nb / ms / 1e6,
                        "ok": bool(torch.equal(o, a.t()))})
            print(json.dumps(res[-1]), flush=True)
    _lib.tune("transpose.scalar_ctas", 0)
    _lib.tune("transpose.scalar_tile", 0)
    del a, o
    torch.cuda.empty_cache()
os.makedirs("gpurun_out", exist_ok=True)
json.dump(res, open("gpurun_out/tune_scalar_big.json", "w"), indent=1)
