"""Per-launch floor inside a CUDA graph: tiny reductions / transposes (all in L2)
vs an empty torch kernel, to split the small-size cost into launch + fixed chain."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2605_13864_b200 as b2  # noqa: E402
from paper_2605_13864_b200 import _lib  # noqa: E402


def graph_us(fn, K=200):
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(K):
            fn()
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


res = {}
z = torch.zeros(1, device="cuda")
res["torch add_ 1 elem"] = graph_us(lambda: z.add_(1))
for logn in [4, 10, 14, 18]:
    x = torch.rand(1 << logn, device="cuda")
    r = torch.empty(1, device="cuda")
    res[f"reduce f32 2^{logn}"] = graph_us(lambda: b2.reduce_sum(x, out=r))
    for cps in [1, 2, 4]:
        _lib.tune("reduce.ctas_per_sm", cps)
        res[f"reduce f32 2^{logn} cps={cps}"] = graph_us(lambda: b2.reduce_sum(x, out=r))
    _lib.tune("reduce.ctas_per_sm", 0)
for n in [32, 256, 1024]:
    a = torch.rand((n, n), device="cuda")
    o = torch.empty_like(a)
    res[f"transpose f32 {n}^2"] = graph_us(lambda: b2.transpose(a, o))
for k, v in res.items():
    print(f"{k:32s} {v:7.2f} us")
os.makedirs("gpurun_out", exist_ok=True)
json.dump(res, open("gpurun_out/floor_probe.json", "w"), indent=1)
