"""Generated kernels with and without the launch-time bounds proof
(B2K_CODEGEN_PROVE=0 forces the checked instantiation): kernel-only GB/s of A.4,
its 64x64-tile variant and A.5 at 8192^2 / 2^26, results compared bit for bit."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2605_13864_b200 as b2  # noqa: E402
from paper_2605_13864_b200 import codegen  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def prog(name):
    with open(os.path.join(ROOT, "tests", "golden", "programs", name)) as f:
        return b2.parse_program(f.read(), name)


def run(name, entry, inputs, prove, reps=7):
    os.environ["B2K_CODEGEN_PROVE"] = "1" if prove else "0"
    p = prog(name)
    c = codegen.compile_fn(p.fn(entry))
    ts, ret = [], None
    for _ in range(reps):
        ret, _ = b2.run_program(p, entry, inputs, backend="codegen")
        ts.append(c.kernel_ms())
    return [statistics.median(t[k] for t in ts[2:]) for k in range(c.n_kernels)], c.kernel_unchecked(), ret


rng = np.random.default_rng(0)
N = 8192
a = rng.uniform(-1, 1, (N, N)).astype(np.float32)
res = []
for name in ["transpose_gpu.optc", "transpose_gpu_t64.optc"]:
    outs = {}
    for prove in (False, True):
        out = np.zeros(N * N, np.float32)
        ms, unchecked, _ = run(name, "transpose", {"in": b2.Array.from_numpy(a.reshape(-1)),
                                                   "out": b2.Array.from_numpy(out), "W": N, "H": N}, prove)
        outs[prove] = out
        res.append({"program": name, "prove": prove, "unchecked": unchecked, "ms": ms[0],
                    "GBps": 2 * N * N * 4 / ms[0] / 1e6})
        print(json.dumps(res[-1]), flush=True)
    assert np.array_equal(outs[False], outs[True]) and np.array_equal(outs[True].reshape(N, N), a.T)
x = rng.uniform(-1, 1, 1 << 26).astype(np.float32)
rets = {}
for prove in (False, True):
    ms, unchecked, ret = run("reduce_tree_f32.optc", "reduce", {"arr": b2.Array.from_numpy(x), "N": x.size}, prove)
    rets[prove] = ret
    nb = x.size * 4 + (x.size // 512) * 4
    res.append({"program": "reduce_tree_f32.optc", "prove": prove, "unchecked": unchecked, "ms": ms[0],
                "GBps": nb / ms[0] / 1e6})
    print(json.dumps(res[-1]), flush=True)
assert rets[False] == rets[True]
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
json.dump(res, open(os.path.join(ROOT, "gpurun_out", "codegen_prove_ab.json"), "w"), indent=1)
