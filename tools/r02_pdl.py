"""Programmatic dependent launch (launch.pdl) A/B on one box, interleaved:
latency-bound back-to-back launches (BASELINE C1 1024^2 transpose, C2 fp32 2^24
sum, paper 4096^2 transpose; CUDA graph over rotating inputs >= 3x L2, per-launch
time) and the full bench step (C4 transpose + C3 sum in one graph)."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2605_13864_b200 as b2  # noqa: E402
from paper_2605_13864_b200 import _lib  # noqa: E402

L2 = 126 * 1024 * 1024


def graph_per_launch(fns, K):
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
    for i in range(8):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        if i >= 2:
            ts.append(e0.elapsed_time(e1) / K)
    del g
    return statistics.median(ts)


cases = {}
for n in (1024, 4096):
    R = max(2, -(-3 * L2 // (2 * n * n * 4)))
    a = [torch.rand((n, n), device="cuda") for _ in range(R)]
    o = [torch.empty_like(a[0]) for _ in range(R)]
    cases[f"transpose_{n}sq_f32"] = (2 * n * n * 4, [(lambda i=i, a=a, o=o: b2.transpose(a[i], o[i])) for i in range(R)], R)
n = 1 << 24
R = max(2, -(-3 * L2 // (n * 4)))
xs = [torch.rand(n, device="cuda") for _ in range(R)]
rs = [torch.empty(1, device="cuda") for _ in range(R)]
cases["reduce_2^24_f32"] = (n * 4 + 4, [(lambda i=i: b2.reduce_sum(xs[i], out=rs[i])) for i in range(R)], R)
A = torch.rand((32768, 32768), device="cuda")
O = torch.empty_like(A)
X = torch.randint(-2**31, 2**31 - 1, (1 << 30,), device="cuda", dtype=torch.int32)
P = torch.zeros(1, dtype=torch.int64, device="cuda")
cases["bench_step"] = (2 * 32768 * 32768 * 4 + (1 << 30) * 4 + 8,
                       [lambda: (b2.transpose(A, O), b2.reduce_sum(X, out=P))], 1)
for rnd in range(2):
    for pdl in (0, 1):
        _lib.tune("launch.pdl", pdl)
        rec = {"pdl": pdl, "round": rnd}
        for name, (nb, fns, R) in cases.items():
            ms = graph_per_launch(fns, 20 if name == "bench_step" else max(2 * R, 64))
            rec[name] = {"us": ms * 1e3, "GBps": nb / ms / 1e6}
        print(json.dumps(rec), flush=True)
_lib.tune("launch.pdl", 0)
assert torch.equal(O, A.t())
