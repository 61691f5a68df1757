"""BASELINE config C5 size sweep on one B200: reductions 2^10 .. 2^32 (fp32,
int32) and odd / non-square transposes (bf16, fp32, fp64), each checked
against the CPU oracle, timed with CUDA events (median of REPS after warm-up,
L2 flushed by a 252 MB read pass (clean lines, no write-back inside the timed
kernel) before every launch when the working set is
smaller than 4x L2). Every case is also timed pipelined: one CUDA graph of
back-to-back launches over R >= 2 rotating copies totalling >= 3x L2, which
removes the ~6 us CUDA-event floor and includes the write-back of the previous
launch's dirty lines, i.e. the steady state of a stream of launches. Also times the in-step interference experiment
(transpose and reduce alternating vs. isolated vs. CUDA-graph captured).

usage: python tools/sweep_c5.py  -> gpurun_out/sweep_c5.json
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
from oracle import oracle  # noqa: E402  (checker only)

L2 = 126 * 1024 * 1024
REPS = 100  # >= 100 timed reps, median and best reported
dev = torch.device("cuda", 0)
flush = torch.ones(2 * L2 // 4, dtype=torch.float32, device=dev)
results = []


def timeit(fn, nbytes, reps=REPS):
    do_flush = nbytes < 4 * L2
    for _ in range(3):
        fn()
    ts = []
    for i in range(reps):
        if do_flush:
            flush.sum()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts), min(ts), do_flush


def pipelined(make, nbytes, K_min=8):
    """Per-launch time inside one CUDA graph of back-to-back launches over R rotating
    copies (inputs + outputs) of the case; cold when R * nbytes >= 3x L2 (R <= 64)."""
    R = int(min(64, max(2, -(-3 * L2 // max(nbytes, 1)))))
    fns = [make() for _ in range(R)]
    K = max(2 * R, K_min)
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        for f in fns:
            f()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        for i in range(K):
            fns[i % R]()
    ts = []
    for i in range(7):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        if i >= 2:
            ts.append(e0.elapsed_time(e1) / K)
    del g, fns
    torch.cuda.empty_cache()
    return statistics.median(ts), R, R * nbytes >= 3 * L2


def rec(**kw):
    results.append(kw)
    print(json.dumps(kw), flush=True)


def reductions():
    for k in list(range(10, 31, 2)) + [31, 32]:
        n = 1 << k
        for dt in ("int32", "float32"):
            if dt == "int32":
                x = torch.randint(-2**31, 2**31, (n,), device=dev, dtype=torch.int64).to(torch.int32) \
                    if k <= 30 else torch.empty(n, dtype=torch.int32, device=dev).random_()
                out = torch.empty(1, dtype=torch.int64, device=dev)
            else:
                x = torch.empty(n, dtype=torch.float32, device=dev).uniform_(-1, 1)
                out = torch.empty(1, dtype=torch.float32, device=dev)
            nbytes = n * 4 + out.element_size()
            ms, best, fl = timeit(lambda: b2.reduce_sum(x, out=out), nbytes)
            got = out.item()
            xh = x.cpu().numpy()
            if dt == "int32":
                ok = int(got) == oracle.reduce_i32(xh)
            else:
                exact, absum = oracle.sum_f64(xh)
                ok = abs(got - exact) <= oracle.f32_tolerance(n, exact, absum)

            def make(x=x, out=out):
                xc, oc = x.clone(), torch.empty_like(out)
                return lambda: b2.reduce_sum(xc, out=oc)
            pms, R, cold = pipelined(make, nbytes)
            extra = dict(us_pipelined=pms * 1e3, GBps_pipelined=nbytes / pms / 1e6, rotating=R,
                         pipelined_cold=cold)
            rec(what="reduce", dtype=dt, n=n, log2n=k, ms=ms, us=ms * 1e3, GBps=nbytes / ms / 1e6, best_us=best * 1e3,
                GBps_best=nbytes / best / 1e6,
                l2_flushed=fl, parity=bool(ok), **extra)
            del x, xh
            torch.cuda.empty_cache()


def transposes():
    shapes = [(1, 1), (1, 1 << 20), (1 << 20, 1), (33, 65), (1023, 1025), (4097, 8191), (4096, 4096),
              (8192, 16384)]
    for dtn in ("bfloat16", "float32", "float64"):
        dt = getattr(torch, dtn)
        iv = {torch.bfloat16: torch.int16, torch.float32: torch.int32, torch.float64: torch.int64}[dt]
        for (H, W) in shapes:
            a = torch.empty((H, W), device=dev, dtype=dt).uniform_(-1, 1)
            o = torch.empty((W, H), device=dev, dtype=dt)
            nbytes = 2 * a.numel() * a.element_size()
            ms, best, fl = timeit(lambda: b2.transpose(a, o), nbytes)
            ok = np.array_equal(o.view(iv).cpu().numpy(), oracle.transpose(a.view(iv).cpu().numpy()))
            extra = {}
            if nbytes:
                def make(a=a):
                    ac, oc = a.clone(), torch.empty((a.shape[1], a.shape[0]), device=dev, dtype=a.dtype)
                    return lambda: b2.transpose(ac, oc)
                pms, R, cold = pipelined(make, nbytes)
                extra = dict(us_pipelined=pms * 1e3, GBps_pipelined=nbytes / pms / 1e6, rotating=R,
                             pipelined_cold=cold)
            rec(what="transpose", dtype=dtn, shape=[H, W], ms=ms, us=ms * 1e3, GBps=nbytes / ms / 1e6,
                best_us=best * 1e3, GBps_best=nbytes / best / 1e6,
                l2_flushed=fl, parity=bool(ok), **extra)
            del a, o
    torch.cuda.empty_cache()


def interference():
    a = torch.empty((32768, 32768), device=dev).uniform_()
    o = torch.empty_like(a)
    x = torch.randint(-2**31, 2**31, (1 << 30,), device=dev, dtype=torch.int64).to(torch.int32)
    r = torch.empty(1, dtype=torch.int64, device=dev)

    def step():
        b2.transpose(a, o)
        b2.reduce_sum(x, out=r)

    def timed(fn, reps=20):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps

    rec(what="interference", mode="transpose_only", ms=timed(lambda: b2.transpose(a, o)))
    rec(what="interference", mode="reduce_only", ms=timed(lambda: b2.reduce_sum(x, out=r)))
    rec(what="interference", mode="alternating_step", ms=timed(step))
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        step()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        step()
    rec(what="interference", mode="graph_step", ms=timed(g.replay))


if __name__ == "__main__":
    which = sys.argv[1:] or ["interference", "transposes", "reductions"]
    for w in which:
        globals()[w]()
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "sweep_c5.json"), "w") as f:
        json.dump(results, f, indent=1)
