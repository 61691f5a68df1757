"""Sweep the libb200k performance knobs on the GPU (CUDA-event timing, median of
REPS launches after warm-up; inputs far larger than L2). Also times torch's own
copy_/sum on the same box as a same-hardware reference point.

usage: python tools/tune.py [--quick]   -> prints JSON lines, writes gpurun_out/tune.json
"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2605_13864_b200 as b2  # noqa: E402
from paper_2605_13864_b200 import _lib  # noqa: E402

REPS = 15
results = []


def timeit(fn, reps=REPS, warm=3):
    for _ in range(warm):
        fn()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts), min(ts)


def rec(**kw):
    results.append(kw)
    print(json.dumps(kw), flush=True)


def main():
    quick = "--quick" in sys.argv
    dev = torch.device("cuda", 0)
    # same-box ceilings
    src = torch.empty(1 << 30, dtype=torch.float32, device=dev).uniform_()
    dst = torch.empty_like(src)
    med, best = timeit(lambda: dst.copy_(src))
    rec(what="torch_copy_4GiB", ms=med, GBps=2 * src.numel() * 4 / med / 1e6, best_GBps=2 * src.numel() * 4 / best / 1e6)
    del dst
    xi = torch.randint(-2**31, 2**31, (1 << 30,), device=dev, dtype=torch.int64).to(torch.int32)
    med, best = timeit(lambda: xi.sum(dtype=torch.int64))
    rec(what="torch_sum_int32_2^30", ms=med, GBps=xi.numel() * 4 / med / 1e6)
    r = torch.empty(1, dtype=torch.int64, device=dev)
    for var in ([0, 1, 2, 3, 4] if not quick else [0]):
        for cps in ([0, 1, 2] if var == 0 else [0]):
            _lib.tune("reduce.variant", var)
            _lib.tune("reduce.ctas_per_sm", cps)
            med, best = timeit(lambda: b2.reduce_sum(xi, out=r))
            rec(what="reduce_i32_2^30", variant=var, ctas_per_sm=cps, ms=med,
                GBps=xi.numel() * 4 / med / 1e6, best_GBps=xi.numel() * 4 / best / 1e6)
    _lib.tune("reduce.variant", 0)
    _lib.tune("reduce.ctas_per_sm", 0)
    del xi
    xf = src[: 1 << 30]
    rf = torch.empty(1, device=dev)
    med, _ = timeit(lambda: b2.reduce_sum(xf, out=rf))
    rec(what="reduce_f32_2^30", ms=med, GBps=xf.numel() * 4 / med / 1e6)
    del src, xf

    configs = [("float32", 32768, 32768), ("bfloat16", 32768, 65536), ("float64", 16384, 32768)]
    for dtn, R, C in configs:
        dt = getattr(torch, dtn)
        a = torch.empty((R, C), device=dev, dtype=dt).uniform_() if dt.is_floating_point else None
        o = torch.empty((C, R), device=dev, dtype=dt)
        nbytes = 2 * a.numel() * a.element_size()
        variants = [0, 1, 2] if not quick else [0]
        groups = [1, 2, 4, 8, 16, 32] if not quick else [1, 8]
        for var in variants:
            for grp in groups:
                _lib.tune("transpose.variant", var)
                _lib.tune("transpose.group", grp)
                med, best = timeit(lambda: b2.transpose(a, o))
                rec(what=f"transpose_{dtn}_{R}x{C}", variant=var, group=grp, ms=med,
                    GBps=nbytes / med / 1e6, best_GBps=nbytes / best / 1e6)
        for cps in [1, 2, 3, 4]:
            _lib.tune("transpose.variant", 0)
            _lib.tune("transpose.group", 1)
            _lib.tune("transpose.ctas_per_sm", cps)
            med, best = timeit(lambda: b2.transpose(a, o))
            rec(what=f"transpose_{dtn}_{R}x{C}", variant=0, group=1, ctas_per_sm=cps, ms=med,
                GBps=nbytes / med / 1e6)
        _lib.tune("transpose.ctas_per_sm", 0)
        # correctness spot check of the last configuration
        torch.cuda.synchronize()
        assert torch.equal(o[:128, :128], a[:128, :128].t())
        med, _ = timeit(lambda: o.copy_(a.t()))
        rec(what=f"torch_transpose_copy_{dtn}_{R}x{C}", ms=med, GBps=nbytes / med / 1e6)
        del a, o
        torch.cuda.empty_cache()
    os.makedirs("gpurun_out", exist_ok=True)
    with open("gpurun_out/tune.json", "w") as f:
        json.dump(results, f, indent=1)


if __name__ == "__main__":
    main()
