"""One bf16 32768x65536 and one fp32 32768^2 transpose launch each (for ncu)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2605_13864_b200 as b2  # noqa: E402

for dt, (r, c) in [(torch.bfloat16, (32768, 65536)), (torch.float32, (32768, 32768))]:
    a = torch.empty((r, c), device="cuda", dtype=dt).uniform_()
    o = torch.empty((c, r), device="cuda", dtype=dt)
    for _ in range(3):
        b2.transpose(a, o)
    torch.cuda.synchronize()
    del a, o
