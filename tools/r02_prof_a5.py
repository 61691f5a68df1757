"""One generated A.5 launch (2^26 fp32, check-free, default coarsening / index type)
for ncu: python tools/r02_prof_a5.py  (run under ncu -k regex:b2g_kernel)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import paper_2605_13864_b200 as b2  # noqa: E402
from paper_2605_13864_b200 import _lib, codegen  # noqa: E402

_lib.tune("codegen.pipe_kb", 0)
name = sys.argv[1] if len(sys.argv) > 1 else "reduce_tree_f32.optc"
with open(os.path.join(ROOT, "tests", "golden", "programs", name)) as f:
    p = b2.parse_program(f.read(), name)
if "reduce" in name:
    x = np.random.default_rng(0).uniform(-1, 1, 1 << 26).astype(np.float32)
    b2.run_program(p, "reduce", {"arr": b2.Array.from_numpy(x), "N": x.size}, backend="codegen")
    c = codegen.compile_fn(p.fn("reduce"))
else:
    N = 8192
    a = np.random.default_rng(0).uniform(-1, 1, (N, N)).astype(np.float32)
    o = np.zeros(N * N, np.float32)
    b2.run_program(p, "transpose", {"in": b2.Array.from_numpy(a.reshape(-1)), "out": b2.Array.from_numpy(o),
                                    "W": N, "H": N}, backend="codegen")
    c = codegen.compile_fn(p.fn("transpose"))
print("coarsen", c.kernel_coarsen(), "ix32", c.kernel_ix32(), "ms", c.kernel_ms())
