"""How much do the generated kernels' interpreter checks cost? Times the
generated A.4 / A.5 kernels as emitted, and with the per-access bounds checks
compiled out (probe only: the product never drops them unproven)."""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import paper_2605_13864_b200 as b2  # noqa: E402
from paper_2605_13864_b200 import codegen  # noqa: E402

CHK = "if (ix < 0 || ix >= d) { b2_flag(f, B2E_OOB, ix, d); return false; }"
orig = codegen.generate
res = []


def run(name, entry, inputs, nbytes, unchecked):
    codegen.generate = (lambda fn: orig(fn).replace(CHK, "")) if unchecked else orig
    codegen._loaded.clear()
    with open(os.path.join(ROOT, "tests", "golden", "programs", name)) as f:
        p = b2.parse_program(f.read(), name)
    c = codegen.compile_fn(p.fn(entry))
    ts = []
    for _ in range(7):
        b2.run_program(p, entry, inputs, backend="codegen")
        ts.append(c.kernel_ms()[0])
    ms = statistics.median(ts[2:])
    res.append({"program": name, "unchecked": unchecked, "ms": ms, "GBps": nbytes / ms / 1e6})
    print(json.dumps(res[-1]), flush=True)


rng = np.random.default_rng(0)
for N in [4096, 16384]:
    a = rng.uniform(-1, 1, (N, N)).astype(np.float32)
    out = np.zeros(N * N, np.float32)
    for unchecked in (False, True):
        for name in ["transpose_gpu.optc", "transpose_gpu_t64.optc"]:
            run(name, "transpose", {"in": b2.Array.from_numpy(a.reshape(-1)), "out": b2.Array.from_numpy(out),
                                    "W": N, "H": N}, 2 * N * N * 4, unchecked)
            assert np.array_equal(out.reshape(N, N), a.T)
x = rng.uniform(-1, 1, 1 << 26).astype(np.float32)
for unchecked in (False, True):
    run("reduce_tree_f32.optc", "reduce", {"arr": b2.Array.from_numpy(x), "N": x.size}, x.size * 4, unchecked)
codegen.generate = orig
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
json.dump(res, open(os.path.join(ROOT, "gpurun_out", "codegen_checks.json"), "w"), indent=1)
