"""A.5 tree order on the hand-written tree_kernel<B> (partials only, device entry)
vs the plain single-pass sum, per launch in a CUDA graph over rotating inputs (>= 3x
L2): GB/s at 2^24 / 2^26 / 2^28 fp32 for B = 512 (A.5) and 64 / 2048."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2605_13864_b200 as b2  # noqa: E402


def graph_us(fns, K=60):
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for f in fns:
            f()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for i in range(K):
            fns[i % len(fns)]()
    ts = []
    for i in range(7):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        if i >= 2:
            ts.append(e0.elapsed_time(e1) * 1000 / K)
    return statistics.median(ts)


for lg in (24, 26, 28):
    n = 1 << lg
    R = max(2, -(-3 * 126 * 2**20 // (4 * n)))
    xs = [torch.empty(n, device="cuda").uniform_() for _ in range(R)]
    rec = {"n": f"2^{lg}", "R": R}
    for B in (64, 512, 2048):
        parts = [torch.empty(n // B, device="cuda") for _ in range(R)]
        us = graph_us([lambda i=i: b2.reduce_tree512_partials(xs[i], parts[i]) if B == 512 else
                       b2.ops.reduce_tree_partials(xs[i], B, parts[i]) for i in range(R)])
        rec[f"tree{B}_GBps"] = round((4 * n + 4 * n // B) / us / 1e3, 1)
    outs = [torch.empty(1, device="cuda") for _ in range(R)]
    us = graph_us([lambda i=i: b2.reduce_sum(xs[i], out=outs[i]) for i in range(R)])
    rec["sum_GBps"] = round((4 * n + 4) / us / 1e3, 1)
    print(json.dumps(rec), flush=True)
    del xs
    torch.cuda.empty_cache()
