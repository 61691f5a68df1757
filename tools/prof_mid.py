"""Mid-size transposes for ncu: bf16 / fp32 8192x16384 and bf16 32768x65536 (one launch each)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2605_13864_b200 as b2  # noqa: E402

for dt, (R, C) in [(torch.bfloat16, (8192, 16384)), (torch.float32, (8192, 16384)), (torch.bfloat16, (32768, 65536))]:
    a = torch.empty((R, C), device="cuda", dtype=dt).uniform_()
    o = torch.empty((C, R), device="cuda", dtype=dt)
    b2.transpose(a, o)
    torch.cuda.synchronize()
    del a, o
    torch.cuda.empty_cache()
