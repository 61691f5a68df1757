"""Kernel-only GB/s of the GENERATED kernels (A.4, its 64x64-tile variant, A.5) at
8192^2 / 2^26 with thread coarsening off / 2 / 4 / 8 (codegen.coarsen) and block packing
(codegen.pack), one launch per
call (codegen.pipe_kb = 0: no chunking, so kernel_ms is the whole kernel), results
compared bit for bit across settings and against numpy."""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import paper_2605_13864_b200 as b2  # noqa: E402
from paper_2605_13864_b200 import _lib, codegen  # noqa: E402


def prog(name):
    with open(os.path.join(ROOT, "tests", "golden", "programs", name)) as f:
        return b2.parse_program(f.read(), name)


def run(p, entry, inputs, reps=7):
    c = codegen.compile_fn(p.fn(entry))
    ts, ret = [], None
    for _ in range(reps):
        ret, _ = b2.run_program(p, entry, inputs, backend="codegen")
        ts.append(c.kernel_ms()[0])
    return statistics.median(ts[2:]), (c.kernel_coarsen()[0], c.kernel_pack()[0]), c.kernel_unchecked()[0], ret


_lib.tune("codegen.pipe_kb", 0)
rng = np.random.default_rng(0)
N = 8192
a = rng.uniform(-1, 1, (N, N)).astype(np.float32)
x = rng.uniform(-1, 1, 1 << 26).astype(np.float32)
SETTINGS = [(1, 1), (2, 1), (4, 1), (8, 1), (8, 4)]  # (codegen.coarsen, codegen.pack) caps
if len(sys.argv) > 1:
    SETTINGS = [tuple(int(v) for v in s.split("x")) for s in sys.argv[1].split(",")]
for rnd in range(2):
    for co, pk in SETTINGS:
        _lib.tune("codegen.coarsen", co)
        _lib.tune("codegen.pack", pk)
        for name in ("transpose_gpu.optc", "transpose_gpu_t64.optc"):
            out = np.zeros(N * N, np.float32)
            ms, got_co, unchecked, _ = run(prog(name), "transpose", {"in": b2.Array.from_numpy(a.reshape(-1)),
                                                                    "out": b2.Array.from_numpy(out), "W": N, "H": N})
            assert np.array_equal(out.reshape(N, N), a.T)
            print(json.dumps({"program": name, "coarsen_max": co, "pack_max": pk, "coarsen_pack": got_co, "unchecked": unchecked,
                              "ms": ms, "GBps": 2 * N * N * 4 / ms / 1e6}), flush=True)
        ms, got_co, unchecked, ret = run(prog("reduce_tree_f32.optc"), "reduce",
                                         {"arr": b2.Array.from_numpy(x), "N": x.size})
        nb = x.size * 4 + (x.size // 512) * 4
        print(json.dumps({"program": "reduce_tree_f32.optc", "coarsen_max": co, "pack_max": pk, "coarsen_pack": got_co,
                          "unchecked": unchecked, "ms": ms, "GBps": nb / ms / 1e6,
                          "result_bits": int(np.float32(ret).view(np.uint32))}), flush=True)
