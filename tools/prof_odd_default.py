"""One odd-pitch transpose through the default dispatch, for ncu: argv dtype rows cols."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2605_13864_b200 as b2  # noqa: E402

dt = {"bf16": torch.bfloat16, "f32": torch.float32, "f64": torch.float64}[sys.argv[1]]
R, C = int(sys.argv[2]), int(sys.argv[3])
a = torch.empty((R, C), device="cuda", dtype=dt)
o = torch.empty((C, R), device="cuda", dtype=dt)
for _ in range(3):
    b2.transpose(a, o)
torch.cuda.synchronize()
