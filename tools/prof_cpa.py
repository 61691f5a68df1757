"""One C4 (fp32 32768^2) transpose with the cp.async path (auto, or variant argv[1])
or the LDG path ("ldg"), for ncu captures; argv: variant dtype [rows cols]."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2605_13864_b200 as b2  # noqa: E402
from paper_2605_13864_b200 import _lib  # noqa: E402

v = sys.argv[1] if len(sys.argv) > 1 else "0"
if v == "ldg":
    _lib.tune("transpose.cpa", 0)
elif v != "auto":
    _lib.tune("transpose.cpa", 2)
    _lib.tune("transpose.cpa_variant", int(v))
dt = {"f32": torch.float32, "bf16": torch.bfloat16, "f64": torch.float64}[sys.argv[2] if len(sys.argv) > 2 else "f32"]
R, C = (32768, 32768) if dt == torch.float32 else ((32768, 65536) if dt == torch.bfloat16 else (16384, 32768))
if len(sys.argv) > 4:
    R, C = int(sys.argv[3]), int(sys.argv[4])
a = torch.empty((R, C), device="cuda", dtype=dt)
o = torch.empty((C, R), device="cuda", dtype=dt)
for _ in range(3):
    b2.transpose(a, o)
torch.cuda.synchronize()
