"""Isolated reduce GB/s (2^30 int32 / fp32) for the current B2K_TUNE setting."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2605_13864_b200 as b2  # noqa: E402

n = 1 << 30
xi = torch.randint(-2**31, 2**31, (n,), device="cuda", dtype=torch.int64).to(torch.int32)
xf = torch.rand(n, device="cuda")
o = {}
for name, x in [("int32", xi), ("float32", xf)]:
    r = torch.empty(1, dtype=torch.int64 if name == "int32" else torch.float32, device="cuda")
    for _ in range(3):
        b2.reduce_sum(x, out=r)
    ts = []
    for _ in range(20):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        b2.reduce_sum(x, out=r)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    o[name] = round((4 * n + 8) / statistics.median(ts) / 1e6)
print(os.environ.get("B2K_TUNE", ""), json.dumps(o))
