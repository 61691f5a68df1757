"""Time breakdown of a generated-code run on pageable vs pinned host arrays."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2605_13864_b200 as b2  # noqa: E402
from paper_2605_13864_b200 import codegen  # noqa: E402

N = 8192
with open("tests/golden/programs/transpose_gpu.optc") as f:
    p = b2.parse_program(f.read())
c = codegen.compile_fn(p.fn("transpose"))
big = np.random.default_rng(0).uniform(-1, 1, N * N).astype(np.float32)
for label in ("pageable", "pinned", "pageable"):
    if label == "pinned":
        src = torch.from_numpy(big).pin_memory().numpy()
        dst = torch.zeros(N * N).pin_memory().numpy()
    else:
        src = big.copy()
        dst = np.zeros(N * N, np.float32)
    inputs = {"in": b2.Array.from_numpy(src), "out": b2.Array.from_numpy(dst), "W": N, "H": N}
    for rep in range(3):
        t0 = time.perf_counter()
        b2.run_program(p, "transpose", inputs, backend="codegen")
        t1 = time.perf_counter()
        print(label, rep, f"{(t1-t0)*1e3:.1f} ms", "kernel ms", [round(x, 3) for x in c.kernel_ms()], flush=True)
