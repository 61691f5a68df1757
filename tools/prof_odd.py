"""ncu driver: odd-pitch transposes through the funnel path (transpose.any=1) and
the padded scalar path (transpose.any=0)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2605_13864_b200 as b2  # noqa: E402
from paper_2605_13864_b200 import _lib  # noqa: E402

dt = getattr(torch, os.environ.get("DTYPE", "float32"))
a = torch.rand((4097, 8191), device="cuda").to(dt)
o = torch.empty((8191, 4097), device="cuda", dtype=dt)
for any_ in (1, 0):
    _lib.tune("transpose.any", any_)
    for _ in range(3):
        b2.transpose(a, o)
torch.cuda.synchronize()
print("ok")
