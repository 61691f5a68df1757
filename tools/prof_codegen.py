"""One generated A.4 launch at 8192^2 (for ncu)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2605_13864_b200 as b2  # noqa: E402

N = 8192
a = np.random.default_rng(0).uniform(-1, 1, (N, N)).astype(np.float32)
out = np.zeros(N * N, np.float32)
p = b2.parse_program(b2.programs.TRANSPOSE_GPU)
for _ in range(2):
    b2.run_program(p, "transpose", {"in": b2.Array.from_numpy(a.reshape(-1)), "out": b2.Array.from_numpy(out),
                                    "W": N, "H": N}, backend="codegen")
