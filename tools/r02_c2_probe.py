"""C2 (fp32 2^24 sum) per-launch time inside a CUDA graph over rotating inputs (6 x
64 MB >= 3x L2): ours vs torch.sum (CUB / ATen reduction) and a plain 64-MB device
copy, to separate the fixed cost of a launch from what the reduction adds."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2605_13864_b200 as b2  # noqa: E402


def graph_us(fns, K=120):
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
    for i in range(9):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        if i >= 2:
            ts.append(e0.elapsed_time(e1) * 1000 / K)
    return statistics.median(ts)


R = 6
xs = [torch.empty(1 << 24, device="cuda").uniform_() for _ in range(R)]
xi = [torch.randint(-2**31, 2**31, (1 << 24,), device="cuda", dtype=torch.int32) for _ in range(R)]
outs = [torch.empty(1, device="cuda", dtype=torch.float32) for _ in range(R)]
outi = [torch.empty(1, device="cuda", dtype=torch.int64) for _ in range(R)]
half = [torch.empty(1 << 23, device="cuda") for _ in range(R)]
res = {}
for rnd in range(2):
    res.setdefault("b2_f32", []).append(graph_us([lambda i=i: b2.reduce_sum(xs[i], out=outs[i]) for i in range(R)]))
    res.setdefault("b2_i32", []).append(graph_us([lambda i=i: b2.reduce_sum(xi[i], out=outi[i]) for i in range(R)]))
    res.setdefault("torch_sum_f32", []).append(graph_us([lambda i=i: torch.sum(xs[i], 0, out=outs[i][0]) for i in range(R)]))
    res.setdefault("torch_sum_i32_to_i64", []).append(
        graph_us([lambda i=i: torch.sum(xi[i], 0, dtype=torch.int64, out=outi[i][0]) for i in range(R)]))
    # a 32-MB -> 32-MB copy moves the same 64 MB of DRAM traffic (read + write)
    res.setdefault("copy_32MB", []).append(graph_us([lambda i=i: half[i].copy_(xs[i][: 1 << 23]) for i in range(R)]))
print(json.dumps({k: [round(v, 2) for v in vs] for k, vs in res.items()}))
