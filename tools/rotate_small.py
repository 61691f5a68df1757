"""Latency-bound cases timed two ways: (1) one launch between CUDA events after a
252 MB read pass (bench.py paper_configs today: includes the ~6 us event floor);
(2) a CUDA graph of back-to-back launches over R rotating input buffers whose
total is >= 3x L2, so no launch finds its input in L2 (the last touch of a
buffer is R-1 launches, >= 2x L2 of traffic, earlier). Parity of each result
is checked against torch."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2605_13864_b200 as b2  # noqa: E402

L2 = 126 * 1024 * 1024
flush = torch.ones(2 * L2 // 4, device="cuda")
res = []


def ev_single(fn, reps=30):
    ts = []
    for i in range(reps + 3):
        flush.sum()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn(0)
        e1.record()
        torch.cuda.synchronize()
        if i >= 3:
            ts.append(e0.elapsed_time(e1))
    return statistics.median(ts) * 1e3


def graph_rot(fn, R, per_graph=None):
    K = per_graph or max(2 * R, 64)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for i in range(R):
            fn(i)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for i in range(K):
            fn(i % R)
    ts = []
    for i in range(8):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        if i >= 2:
            ts.append(e0.elapsed_time(e1) / K)
    return statistics.median(ts) * 1e3


for logn in [20, 22, 24, 26]:
    nb = (1 << logn) * 4
    R = max(2, -(-3 * L2 // nb))
    xs = [torch.rand(1 << logn, device="cuda") for _ in range(R)]
    outs = [torch.empty(1, device="cuda") for _ in range(R)]
    f = lambda i: b2.reduce_sum(xs[i], out=outs[i])  # noqa: E731
    us1 = ev_single(f)
    us2 = graph_rot(f, R)
    ok = all(abs(outs[i].item() - xs[i].double().sum().item()) <= 1e-5 * xs[i].abs().double().sum().item()
             for i in range(R))
    rec = dict(what="reduce f32", log2n=logn, R=R, single_event_us=us1, graph_rotating_us=us2,
               GBps_single=nb / us1 / 1e3, GBps_graph=nb / us2 / 1e3, parity=ok)
    print(json.dumps(rec), flush=True)
    res.append(rec)
    del xs
for n in [1024, 2048, 4096, 8192]:
    nb = n * n * 4
    R = max(2, -(-3 * L2 // (2 * nb)))
    xs = [torch.rand((n, n), device="cuda") for _ in range(R)]
    ys = [torch.empty_like(xs[0]) for _ in range(R)]
    f = lambda i: b2.transpose(xs[i], ys[i])  # noqa: E731
    us1 = ev_single(f)
    us2 = graph_rot(f, R)
    ok = all(torch.equal(ys[i], xs[i].t()) for i in range(R))
    rec = dict(what="transpose f32", n=n, R=R, single_event_us=us1, graph_rotating_us=us2,
               GBps_single=2 * nb / us1 / 1e3, GBps_graph=2 * nb / us2 / 1e3, parity=ok)
    print(json.dumps(rec), flush=True)
    res.append(rec)
    del xs, ys
os.makedirs("gpurun_out", exist_ok=True)
json.dump(res, open("gpurun_out/rotate_small.json", "w"), indent=1)
