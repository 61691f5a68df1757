"""Reduction variants / residency at latency-bound sizes (2^20 .. 2^26, fp32 and
int32), pipelined: CUDA graph over rotating inputs totalling >= 3x L2."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2605_13864_b200 as b2  # noqa: E402
from paper_2605_13864_b200 import _lib  # noqa: E402

L2 = 126 * 1024 * 1024


def graph_us(fns, K):
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        for f in fns:
            f()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        for i in range(K):
            fns[i % len(fns)]()
    ts = []
    for i in range(9):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        if i >= 3:
            ts.append(e0.elapsed_time(e1) / K)
    return statistics.median(ts) * 1e3


for logn in [20, 22, 24, 26]:
    n = 1 << logn
    R = max(2, -(-3 * L2 // (4 * n)))
    for dt in (torch.float32, torch.int32):
        xs = [(torch.rand(n, device="cuda") if dt == torch.float32 else
               torch.randint(-2**31, 2**31 - 1, (n,), device="cuda", dtype=torch.int32)) for _ in range(R)]
        outs = [torch.empty(1, device="cuda", dtype=torch.float32 if dt == torch.float32 else torch.int64)
                for _ in range(R)]
        fns = [(lambda x=x, o=o: b2.reduce_sum(x, out=o)) for x, o in zip(xs, outs)]
        res = []
        for var, cps in [(0, 0), (0, 1), (0, 3), (0, 4), (1, 0), (1, 1), (3, 0), (3, 1), (5, 0), (6, 0), (8, 0),
                         (0, 0)]:
            _lib.tune("reduce.variant", var)
            _lib.tune("reduce.ctas_per_sm", cps)
            res.append(((var, cps), round(graph_us(fns, max(2 * R, 32)), 2)))
        _lib.tune("reduce.variant", 0)
        _lib.tune("reduce.ctas_per_sm", 0)
        print(json.dumps({"log2n": logn, "dtype": str(dt)[6:], "R": R, "us((variant,cps))": res}), flush=True)
        del xs, outs, fns
        torch.cuda.empty_cache()
