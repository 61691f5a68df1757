"""cudaMemcpy2DAsync D2H of transpose column slabs (rows of w bytes at 128 KB
host pitch), alone and concurrent with a contiguous H2D: is the 2-D copy what
keeps the host-buffer transpose (92.6 ms) above the duplex bound (86.8 ms)?"""
import json
import os
import time

import torch
from cuda.bindings import runtime as rt

res = []
n = 1 << 30
d1 = torch.empty(n, dtype=torch.float32, device="cuda")
d2 = torch.empty(n, dtype=torch.float32, device="cuda")
h1 = torch.empty(n, dtype=torch.float32, pin_memory=True)
h2 = torch.empty(n, dtype=torch.float32, pin_memory=True)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
D2H, H2D = rt.cudaMemcpyKind.cudaMemcpyDeviceToHost, rt.cudaMemcpyKind.cudaMemcpyHostToDevice
R, PITCH = 32768, 32768 * 4


def d2h_slabs(w, stream):
    """the whole 4 GiB output as column slabs of w bytes per row"""
    nslab = PITCH // w
    for k in range(nslab):
        src = d2.data_ptr() + k * R * w
        dst = h2.data_ptr() + k * w
        err, = rt.cudaMemcpy2DAsync(dst, PITCH, src, w, w, R, D2H, stream.cuda_stream)
        assert err == rt.cudaError_t.cudaSuccess


def h2d_rows(stream):
    err, = rt.cudaMemcpyAsync(d1.data_ptr(), h1.data_ptr(), 4 * n, H2D, stream.cuda_stream)
    assert err == rt.cudaError_t.cudaSuccess


def wall(fn, reps=2):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps


for w in [1024, 2048, 4096, 8192, 32768]:
    dt = wall(lambda: d2h_slabs(w, s2))
    res.append({"what": f"d2h 2-D, {w} B rows", "GBps": 4 * n / dt / 1e9, "ms": dt * 1e3})
    print(json.dumps(res[-1]), flush=True)
    dt = wall(lambda: (h2d_rows(s1), d2h_slabs(w, s2)))
    res.append({"what": f"h2d contiguous + d2h 2-D {w} B rows, concurrent", "GBps": 8 * n / dt / 1e9,
                "ms": dt * 1e3})
    print(json.dumps(res[-1]), flush=True)
os.makedirs("gpurun_out", exist_ok=True)
json.dump(res, open("gpurun_out/pcie_probe2.json", "w"), indent=1)
