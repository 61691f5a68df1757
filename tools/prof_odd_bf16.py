"""One bf16 / fp16-bit odd-pitch transpose launch (4097x8191), for ncu."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2605_13864_b200 as b2  # noqa: E402

a = torch.empty((4097, 8191), device="cuda", dtype=torch.bfloat16).uniform_()
o = torch.empty((8191, 4097), device="cuda", dtype=torch.bfloat16)
for _ in range(3):
    b2.transpose(a, o)
torch.cuda.synchronize()
