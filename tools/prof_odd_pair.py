"""Odd-pitch transposes for ncu: bf16 and fp32 16385x16383 (large) and 4097x8191,
one launch each after warm-up (ncu -c picks them)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2605_13864_b200 as b2  # noqa: E402

for dt in (torch.bfloat16, torch.float32):
    for (H, W) in [(16385, 16383), (4097, 8191)]:
        a = torch.empty((H, W), device="cuda", dtype=dt).uniform_()
        o = torch.empty((W, H), device="cuda", dtype=dt)
        b2.transpose(a, o)
        torch.cuda.synchronize()
