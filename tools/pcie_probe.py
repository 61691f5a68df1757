"""PCIe probe for the e2e path: what limits the host-buffer transpose?
(1) H2D / D2H alone and concurrently (contiguous, pinned); (2) the 2-D D2H the
transpose pipeline issues (column slabs: 2 KB rows at 128 KB pitch); (3) zero-copy
kernels: libb200k kernels reading / writing pinned host memory directly over PCIe."""
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


def rec(what, nbytes, dt, **kw):
    res.append({"what": what, "GBps": nbytes / dt / 1e9, "ms": dt * 1e3, **kw})
    print(json.dumps(res[-1]), flush=True)


def wall(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps


n = 1 << 30  # 4 GiB
d1 = torch.empty(n, dtype=torch.float32, device="cuda")
d2 = torch.empty(n, dtype=torch.float32, device="cuda")
h1 = torch.empty(n, dtype=torch.float32, pin_memory=True)
h2 = torch.empty(n, dtype=torch.float32, pin_memory=True)
h1.numpy()[:] = 1.0
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
rec("h2d", 4 * n, wall(lambda: d1.copy_(h1, non_blocking=True)))
rec("d2h", 4 * n, wall(lambda: h2.copy_(d2, non_blocking=True)))


def both():
    with torch.cuda.stream(s1):
        d1.copy_(h1, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)


rec("h2d+d2h concurrent (aggregate)", 8 * n, wall(both))
# 2-D D2H: 2 KB rows at 128 KB pitch (the transpose pipeline's column slabs)
R = 32768
for wbytes in [2048, 4096, 8192, 16384]:
    wcols = wbytes // 4
    dsrc = d2[: R * wcols].view(R, wcols)
    hdst = h2.view(R, 32768)[:, :wcols]
    nb = R * wbytes
    reps = 8

    def d2h2():
        for _ in range(reps):
            hdst.copy_(dsrc, non_blocking=True)
    rec(f"d2h 2-D rows of {wbytes} B (pitch 128 KB)", nb * reps, wall(d2h2, 2))
# zero-copy: the reduction kernel reading pinned host memory
x = h1.view(torch.int32)
out = torch.zeros(1, dtype=torch.int64, device="cuda")
L = _lib.lib()


def zc_reduce():
    _lib.check(L.b2_reduce_sum(x.data_ptr(), n, _lib.I32, out.data_ptr(), None, 0, 0,
                               torch.cuda.current_stream().cuda_stream))
rec("zero-copy reduce (kernel reads pinned host)", 4 * n, wall(zc_reduce))
# zero-copy transpose: device input -> pinned host output, and host input -> device output
a = d1.view(32768, 32768)
ho = h2.view(32768, 32768)


def zc_t_out():
    _lib.check(L.b2_transpose(a.data_ptr(), ho.data_ptr(), 32768, 32768, 32768, 32768, _lib.F32, 0,
                              torch.cuda.current_stream().cuda_stream))
rec("zero-copy transpose, output to pinned host", 4 * n, wall(zc_t_out, 2))
hi = h1.view(32768, 32768)
do = d2.view(32768, 32768)


def zc_t_in():
    _lib.check(L.b2_transpose(hi.data_ptr(), do.data_ptr(), 32768, 32768, 32768, 32768, _lib.F32, 0,
                              torch.cuda.current_stream().cuda_stream))
rec("zero-copy transpose, input from pinned host", 4 * n, wall(zc_t_in, 2))


def zc_t_both():
    _lib.check(L.b2_transpose(hi.data_ptr(), ho.data_ptr(), 32768, 32768, 32768, 32768, _lib.F32, 0,
                              torch.cuda.current_stream().cuda_stream))
rec("zero-copy transpose, host -> host (aggregate both directions)", 8 * n, wall(zc_t_both, 2))
os.makedirs("gpurun_out", exist_ok=True)
json.dump(res, open("gpurun_out/pcie_probe.json", "w"), indent=1)
