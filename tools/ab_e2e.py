"""Host-buffer transpose + reduce (pinned, 4 GiB each) for the library in B2K_LIB."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2605_13864_b200 as b2  # noqa: E402
from paper_2605_13864_b200 import _lib  # noqa: E402

R = C = 32768
hin = torch.ones((R, C), dtype=torch.float32).pin_memory()
hout = torch.empty((C, R), dtype=torch.float32).pin_memory()
hx = torch.ones(1 << 30, dtype=torch.int32).pin_memory()
a, o, x = hin.numpy(), hout.numpy(), hx.numpy()
b2.transpose(a, o)
b2.reduce_sum(x)
t0 = time.perf_counter()
for _ in range(4):
    b2.transpose(a, o)
t1 = time.perf_counter()
for _ in range(4):
    b2.reduce_sum(x)
t2 = time.perf_counter()
print(json.dumps({"lib": os.path.basename(_lib.LIB_PATH), "transpose_ms": (t1 - t0) / 4 * 1e3,
                  "reduce_ms": (t2 - t1) / 4 * 1e3}))
