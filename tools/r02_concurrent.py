"""Bench step (C4 transpose + C3 sum) with the two kernels one after the other vs
concurrently on two forked streams, each as one CUDA graph of K steps: ms per step."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2605_13864_b200 as b2  # noqa: E402

dev = torch.device("cuda", 0)
a = torch.rand((32768, 32768), device=dev)
out = torch.empty((32768, 32768), device=dev)
x = torch.randint(-2**31, 2**31, (1 << 30,), device=dev, dtype=torch.int32)
part = torch.empty(1, device=dev, dtype=torch.int64)
K = 20
s0 = torch.cuda.Stream(dev)
s1 = torch.cuda.Stream(dev)
ws = torch.zeros(b2.ops.reduce_ws_bytes(1 << 30, b2.ops.b2_dtype(x)) // 8 + 8, device=dev, dtype=torch.int64)


def seq_step():
    b2.transpose(a, out)
    b2.reduce_sum(x, out=part)


def conc_step():
    main = torch.cuda.current_stream(dev)
    s1.wait_stream(main)
    b2.transpose(a, out)
    with torch.cuda.stream(s1):
        b2.reduce_sum(x, out=part, ws=ws)
    main.wait_stream(s1)


def graph_ms(step):
    with torch.cuda.stream(s0):
        step()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s0):
        for _ in range(K):
            step()
    g.replay()
    torch.cuda.synchronize()
    ts = []
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / K)
    return min(ts)


nb = 2 * 32768 * 32768 * 4 + (1 << 30) * 4 + 8
res = {}
for rnd in range(3):
    for name, fn in (("sequential", seq_step), ("concurrent", conc_step)):
        ms = graph_ms(fn)
        res.setdefault(name, []).append(round(nb / ms / 1e6, 1))
assert torch.equal(out[:64, :64], a[:64, :64].t()) and int(part.item()) == int(x.to(torch.int64).sum().item())
print(json.dumps({"GBps": res}))
