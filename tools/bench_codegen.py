"""Kernel-only effective bandwidth of the GENERATED kernels (codegen.py) for the
paper's own programs on the paper's benchmark sizes: the
A.4 transpose at 4096^2 fp32 and the A.5 tree reduction at 2^24 fp32, plus the
64x64-tile variant. This is the B200 analogue of Table 7.4's "OptiGPU" column
(297.7 / 297.9 GB/s on an RTX 5060); the hand-written kernels are timed beside.

usage: python tools/bench_codegen.py  -> gpurun_out/bench_codegen.json
"""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2605_13864_b200 as b2  # noqa: E402
from paper_2605_13864_b200 import codegen  # noqa: E402

res = []


def prog(name):
    with open(os.path.join(ROOT, "tests", "golden", "programs", name)) as f:
        return b2.parse_program(f.read(), name)


def gen_time(name, entry, inputs, reps=7):
    p = prog(name)
    fn = p.fn(entry)
    c = codegen.compile_fn(fn)
    ts = []
    for _ in range(reps):
        b2.run_program(p, entry, inputs, backend="codegen")
        ts.append(c.kernel_ms())
    return [statistics.median(t[k] for t in ts[2:]) for k in range(c.n_kernels)]


def main():
    rng = np.random.default_rng(0)
    N = 4096
    a = rng.uniform(-1, 1, (N, N)).astype(np.float32)
    out = np.zeros(N * N, np.float32)
    for name in ["transpose_gpu.optc", "transpose_gpu_t64.optc"]:
        ms = gen_time(name, "transpose", {"in": b2.Array.from_numpy(a.reshape(-1)),
                                          "out": b2.Array.from_numpy(out), "W": N, "H": N})
        assert np.array_equal(out.reshape(N, N), a.T)
        res.append({"program": name, "kernel": "generated", "ms": ms[0],
                    "GBps": 2 * N * N * 4 / ms[0] / 1e6, "paper_rtx5060_optigpu_GBps": 297.7})
        print(json.dumps(res[-1]), flush=True)
    x = rng.uniform(-1, 1, 1 << 24).astype(np.float32)
    ms = gen_time("reduce_tree_f32.optc", "reduce", {"arr": b2.Array.from_numpy(x), "N": x.size})
    nb = x.size * 4 + (x.size // 512) * 4
    res.append({"program": "reduce_tree_f32.optc", "kernel": "generated", "ms": ms[0],
                "GBps": nb / ms[0] / 1e6, "paper_rtx5060_optigpu_GBps": 297.9})
    print(json.dumps(res[-1]), flush=True)
    # hand-written kernels on the same sizes (no L2 flush either: same conditions)
    da = torch.from_numpy(a).cuda()
    do = torch.empty_like(da)
    dx = torch.from_numpy(x).cuda()
    parts = torch.empty(x.size // 512, device="cuda")
    for label, fn, nbytes in [("transpose_vec_kernel (A.4 template)", lambda: b2.transpose(da, do), 2 * N * N * 4),
                              ("tree512_kernel (A.5 template)", lambda: b2.reduce_tree512_partials(dx, parts), nb),
                              ("reduce_kernel (single pass)", lambda: b2.reduce_sum(dx), x.size * 4 + 4)]:
        for _ in range(3):
            fn()
        ts = []
        for _ in range(10):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        ms = statistics.median(ts)
        res.append({"program": label, "kernel": "hand-written", "ms": ms, "GBps": nbytes / ms / 1e6})
        print(json.dumps(res[-1]), flush=True)
    # end to end through run_program (host Arrays, generated host code, copy engine)
    import time
    N2 = 8192
    big = rng.uniform(-1, 1, (N2, N2)).astype(np.float32)
    for label, pin in [("pageable", False), ("pinned", True)]:
        src = torch.from_numpy(big.reshape(-1)).pin_memory().numpy() if pin else big.reshape(-1).copy()
        dst = torch.zeros(N2 * N2, dtype=torch.float32).pin_memory().numpy() if pin else np.zeros(N2 * N2, np.float32)
        p = prog("transpose_gpu.optc")
        inputs = {"in": b2.Array.from_numpy(src), "out": b2.Array.from_numpy(dst), "W": N2, "H": N2}
        b2.run_program(p, "transpose", inputs, backend="codegen")
        t0 = time.perf_counter()
        for _ in range(3):
            b2.run_program(p, "transpose", inputs, backend="codegen")
        dt = (time.perf_counter() - t0) / 3
        assert np.array_equal(dst.reshape(N2, N2), big.T)
        res.append({"program": "transpose_gpu.optc e2e " + label, "kernel": "generated + host copies",
                    "ms": dt * 1e3, "GBps": 2 * N2 * N2 * 4 / dt / 1e9,
                    "note": "run_program wall time: H2D + kernel + D2H through b2_copy_h2d/d2h"})
        print(json.dumps(res[-1]), flush=True)
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "bench_codegen.json"), "w") as f:
        json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
