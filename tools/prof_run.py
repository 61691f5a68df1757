"""Minimal driver for ncu: the two hot-path kernels at the bench sizes, a few
launches each (run under `ncu ... python tools/prof_run.py`)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2605_13864_b200 as b2  # noqa: E402

rows = int(os.environ.get("ROWS", 32768))
cols = int(os.environ.get("COLS", 32768))
n = int(os.environ.get("N", 1 << 30))
reps = int(os.environ.get("REPS", 3))
dt = getattr(torch, os.environ.get("DTYPE", "float32"))
a = torch.rand((rows, cols), device="cuda").to(dt)
o = torch.empty((cols, rows), device="cuda", dtype=dt)
x = torch.randint(-2**31, 2**31, (n,), device="cuda", dtype=torch.int64).to(torch.int32)
r = torch.empty(1, dtype=torch.int64, device="cuda")
for _ in range(reps):
    b2.transpose(a, o)
    b2.reduce_sum(x, out=r)
torch.cuda.synchronize()
print("done", int(r.item()))
