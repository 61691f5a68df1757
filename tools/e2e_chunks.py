"""Host pipeline: raw PCIe H2D/D2H bandwidth (pinned, pageable) and the e2e
run_program step at several chunk sizes (host.chunk_mb)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2605_13864_b200 as b2  # noqa: E402
from paper_2605_13864_b200 import _lib  # noqa: E402

res = []
n = 1 << 30
dbuf = torch.empty(n, dtype=torch.float32, device="cuda")
hp = torch.empty(n, dtype=torch.float32, pin_memory=True)
hq = torch.empty(n, dtype=torch.float32)  # pageable
for name, src, dst in [("h2d_pinned", hp, dbuf), ("d2h_pinned", dbuf, hp), ("h2d_pageable", hq, dbuf),
                       ("d2h_pageable", dbuf, hq)]:
    dst.copy_(src)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(3):
        dst.copy_(src)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / 3
    res.append({"what": name, "GBps": n * 4 / dt / 1e9})
    print(json.dumps(res[-1]), flush=True)
del dbuf, hq
rows = cols = 32768
hin = torch.empty((rows, cols), dtype=torch.float32, pin_memory=True)
hin.numpy()[:] = 1.0
hout = torch.empty((cols, rows), dtype=torch.float32, pin_memory=True)
hx = hp.view(torch.int32)
tp = b2.parse_program(b2.programs.TRANSPOSE_NAIVE)
rp = b2.parse_program(b2.programs.REDUCE_NAIVE_INT)
t_in = {"in": b2.Array.from_numpy(hin.numpy()), "out": b2.Array.from_numpy(hout.numpy()), "W": cols, "H": rows}
r_in = {"arr": b2.Array.from_numpy(hx.numpy(), "int"), "N": n}
for mb in [16, 32, 64, 128, 256, 512]:
    _lib.tune("host.chunk_mb", mb)
    b2.run_program(tp, "transpose", t_in)
    b2.run_program(rp, "reduce", r_in)
    t0 = time.perf_counter()
    for _ in range(3):
        b2.run_program(tp, "transpose", t_in)
    t1 = time.perf_counter()
    for _ in range(3):
        b2.run_program(rp, "reduce", r_in)
    t2 = time.perf_counter()
    tt, tr = (t1 - t0) / 3, (t2 - t1) / 3
    step = 2 * rows * cols * 4 + n * 4 + 8
    res.append({"what": "e2e", "chunk_mb": mb, "transpose_ms": tt * 1e3, "reduce_ms": tr * 1e3,
                "e2e_GBps": step / (tt + tr) / 1e9})
    print(json.dumps(res[-1]), flush=True)
# pageable host buffers (staged through the pinned ring + host copy pool)
_lib.tune("host.chunk_mb", 64)
pin_in, pin_out = np.empty((rows, cols), np.float32), np.empty((cols, rows), np.float32)
pin_in[:] = 1.0
px = np.ones(n, np.int32)
t_in = {"in": b2.Array.from_numpy(pin_in), "out": b2.Array.from_numpy(pin_out), "W": cols, "H": rows}
r_in = {"arr": b2.Array.from_numpy(px, "int"), "N": n}
b2.run_program(tp, "transpose", t_in)
b2.run_program(rp, "reduce", r_in)
t0 = time.perf_counter()
for _ in range(3):
    b2.run_program(tp, "transpose", t_in)
t1 = time.perf_counter()
for _ in range(3):
    b2.run_program(rp, "reduce", r_in)
t2 = time.perf_counter()
tt, tr = (t1 - t0) / 3, (t2 - t1) / 3
res.append({"what": "e2e_pageable", "chunk_mb": 64, "transpose_ms": tt * 1e3, "reduce_ms": tr * 1e3,
            "e2e_GBps": (2 * rows * cols * 4 + n * 4 + 8) / (tt + tr) / 1e9})
print(json.dumps(res[-1]), flush=True)
os.makedirs("gpurun_out", exist_ok=True)
json.dump(res, open("gpurun_out/e2e_chunks.json", "w"), indent=1)
