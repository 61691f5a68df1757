"""Odd-pitch transposes: padded scalar tile at several residencies vs the funnel path."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2605_13864_b200 as b2  # noqa: E402
from paper_2605_13864_b200 import _lib  # noqa: E402

res = []
CONFIGS = [("scalar4", 0, 4), ("scalar2", 0, 2), ("scalar3", 0, 3), ("scalar6", 0, 6), ("scalar8", 0, 8),
           ("any", 1, 4)]
for dtn in ("bfloat16", "float32", "float64"):
    dt = getattr(torch, dtn)
    for (H, W) in [(4097, 8191), (8191, 16383), (20001, 3001)]:
        a = torch.rand((H, W), device="cuda").to(dt)
        o = torch.empty((W, H), device="cuda", dtype=dt)
        nb = 2 * a.numel() * a.element_size()
        row = {"dtype": dtn, "shape": [H, W]}
        for name, any_, sc in CONFIGS:
            _lib.tune("transpose.any", any_)
            _lib.tune("transpose.scalar_ctas", sc)
            for _ in range(3):
                b2.transpose(a, o)
            ts = []
            for _ in range(10):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                b2.transpose(a, o)
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            ms = statistics.median(ts)
            row[name] = round(nb / ms / 1e6)
            assert torch.equal(o, a.t())
        res.append(row)
        print(json.dumps(row), flush=True)
os.makedirs("gpurun_out", exist_ok=True)
json.dump(res, open("gpurun_out/odd_compare.json", "w"), indent=1)
