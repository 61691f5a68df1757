"""SURVEY 8(f) rank 4 in numbers: the reference's own programs at FULL C3 / C4
size through the vectorised restatement of its interpreter (oracle/vinterp.py,
one core), checked against the C oracle. (The reference interpreter itself
would need hours and > 40 GiB of Python objects here.)"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import paper_2605_13864_b200 as b2  # noqa: E402
from oracle import oracle, vinterp  # noqa: E402

res = []
n = 1 << 30
x = np.empty(n, dtype=np.int32)
oracle.fill_u32(x.view(np.uint32), 4)
t0 = time.perf_counter()
s, _ = vinterp.run_program(b2.parse_program(b2.programs.REDUCE_NAIVE_INT), "reduce",
                           {"arr": b2.Array([n], x, "int"), "N": n}, as_numpy=True)
dt = time.perf_counter() - t0
res.append({"program": "A.3 int reduce", "n": n, "seconds": dt, "GBps": (4 * n + 8) / dt / 1e9,
            "exact": s == oracle.reduce_i32(x)})
print(json.dumps(res[-1]), flush=True)
del x
R = C = 32768
a = np.empty((R, C), dtype=np.float32)
oracle.fill_u32(a.view(np.uint32).reshape(-1), 3)
a[~np.isfinite(a)] = 0.0
out = np.zeros(R * C, np.float32)
t0 = time.perf_counter()
vinterp.run_program(b2.parse_program(b2.programs.TRANSPOSE_NAIVE), "transpose",
                    {"in": b2.Array([R, C], a.reshape(-1), "float"), "out": b2.Array([C, R], out, "float"),
                     "W": C, "H": R}, as_numpy=True)
dt = time.perf_counter() - t0
ok = np.array_equal(out.reshape(C, R), oracle.transpose(a))
res.append({"program": "A.1 transpose", "shape": [R, C], "seconds": dt, "GBps": 2 * R * C * 4 / dt / 1e9,
            "bit_exact": bool(ok)})
print(json.dumps(res[-1]), flush=True)
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
json.dump(res, open(os.path.join(ROOT, "gpurun_out", "vinterp_fullsize.json"), "w"), indent=1)
