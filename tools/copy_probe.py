"""Probe the copy engine: b2_copy_h2d / b2_copy_d2h on pageable and pinned buffers."""
import ctypes
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2605_13864_b200 import _lib  # noqa: E402

L = _lib.lib()
n = 64 << 20  # floats = 256 MB
d = torch.empty(n, dtype=torch.float32, device="cuda")
print("cpus", os.cpu_count(), flush=True)
for label, h in [("pageable", np.ones(n, np.float32)), ("pinned", torch.ones(n).pin_memory().numpy())]:
    for direction in ("h2d", "d2h"):
        fn = L.b2_copy_h2d if direction == "h2d" else L.b2_copy_d2h
        args = (d.data_ptr(), h.ctypes.data) if direction == "h2d" else (h.ctypes.data, d.data_ptr())
        for rep in range(3):
            t0 = time.perf_counter()
            rc = fn(args[0], args[1], n * 4, 0)
            dt = time.perf_counter() - t0
            print(label, direction, rep, rc, f"{dt*1e3:.1f} ms", f"{n*4/dt/1e9:.1f} GB/s", flush=True)
    t0 = time.perf_counter()
    d.copy_(torch.from_numpy(h))
    torch.cuda.synchronize()
    print(label, "torch h2d", f"{(time.perf_counter()-t0)*1e3:.1f} ms", flush=True)
