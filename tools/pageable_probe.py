"""e2e with PAGEABLE host buffers (plain numpy arrays, how list-based callers of
run_program arrive) at the current B2K_COPY_THREADS setting."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2605_13864_b200 as b2  # noqa: E402

R = C = 32768
a = np.ones((R, C), dtype=np.float32)
o = np.empty((C, R), dtype=np.float32)
x = np.ones(1 << 30, dtype=np.int32)
b2.transpose(a, o)
b2.reduce_sum(x)
t0 = time.perf_counter()
for _ in range(2):
    b2.transpose(a, o)
t1 = time.perf_counter()
for _ in range(2):
    b2.reduce_sum(x)
t2 = time.perf_counter()
print(json.dumps({"threads": os.environ.get("B2K_COPY_THREADS", "default"),
                  "transpose_ms": (t1 - t0) / 2 * 1e3, "reduce_ms": (t2 - t1) / 2 * 1e3,
                  "e2e_GBps": (2 * R * C * 4 + x.size * 4) / ((t2 - t0) / 2) / 1e9}))
