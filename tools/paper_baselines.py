"""The paper's SIMT kernels (tools/paperk/paper_kernels.cu) recompiled for
sm_100a vs the B200 kernels, on the paper's Table 7.4 workloads (4096^2 fp32
transpose, 2^24 fp32 sum; cold L2) and the bench workloads (C4 32768^2, 2^30).

usage: python tools/paper_baselines.py  -> gpurun_out/paper_baselines.json
"""
import ctypes
import json
import os
import statistics
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2605_13864_b200 as b2  # noqa: E402

HERE = os.path.join(ROOT, "tools", "paperk")
SO = os.path.join(HERE, "libpaperk.so")
subprocess.run(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-shared",
                "-Xcompiler", "-fPIC", "-o", SO, os.path.join(HERE, "paper_kernels.cu")], check=True)
PK = ctypes.CDLL(SO)
PK.pk_transpose.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_void_p]
PK.pk_reduce.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p,
                         ctypes.c_void_p]
L2 = 126 * 1024 * 1024
flush = torch.ones(2 * L2 // 4, device="cuda")
res = []


def timeit(fn, cold, reps=15):
    for _ in range(3):
        fn()
    ts = []
    for _ in range(reps):
        if cold:
            flush.sum()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)


def s():
    return torch.cuda.current_stream().cuda_stream


for n in [4096, 32768]:
    a = torch.rand((n, n), device="cuda")
    o = torch.empty_like(a)
    nb = 2 * n * n * 4
    cold = nb < 4 * L2
    for name, fn in [("paper transpose_naive", lambda: PK.pk_transpose(0, a.data_ptr(), o.data_ptr(), n, n, s())),
                     ("paper transpose_tile32 (Listing 3.6 / OptiGPU)",
                      lambda: PK.pk_transpose(1, a.data_ptr(), o.data_ptr(), n, n, s())),
                     ("paper transposeNoBankConflicts (32x33)",
                      lambda: PK.pk_transpose(2, a.data_ptr(), o.data_ptr(), n, n, s())),
                     ("b2 transpose", lambda: b2.transpose(a, o))]:
        ms = timeit(fn, cold)
        ok = bool(torch.equal(o, a.t()))
        o.zero_()
        res.append({"kernel": name, "shape": [n, n], "ms": ms, "GBps": nb / ms / 1e6, "ok": ok, "cold_l2": cold})
        print(json.dumps(res[-1]), flush=True)
    del a, o
for logn in [24, 30]:
    n = 1 << logn
    x = torch.rand(n, device="cuda") - 0.5
    tmp = torch.empty(n // 256 + 64, device="cuda")
    out = torch.empty(1, device="cuda")
    want = x.double().sum().item()
    nb = n * 4
    cold = nb < 4 * L2
    for name, fn in [("paper reduce OptiGPU tree (A.5)", lambda: PK.pk_reduce(0, x.data_ptr(), n, tmp.data_ptr(), out.data_ptr(), s())),
                     ("paper reduce3", lambda: PK.pk_reduce(1, x.data_ptr(), n, tmp.data_ptr(), out.data_ptr(), s())),
                     ("paper reduce6", lambda: PK.pk_reduce(2, x.data_ptr(), n, tmp.data_ptr(), out.data_ptr(), s())),
                     ("b2 reduce_sum", lambda: b2.reduce_sum(x, out=out))]:
        ms = timeit(fn, cold)
        got = out.item()
        res.append({"kernel": name, "n": n, "ms": ms, "GBps": nb / ms / 1e6, "abs_err": abs(got - want),
                    "cold_l2": cold})
        print(json.dumps(res[-1]), flush=True)
    del x, tmp
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
json.dump(res, open(os.path.join(ROOT, "gpurun_out", "paper_baselines.json"), "w"), indent=1)
