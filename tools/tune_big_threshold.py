"""128-KB tiles (transpose.big = 2 forces them) vs the default choice on mid sizes,
pipelined clock (CUDA graph over rotating copies >= 3x L2)."""
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
    for i in range(7):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        if i >= 2:
            ts.append(e0.elapsed_time(e1) / K)
    return statistics.median(ts) * 1e3


for dt in (torch.float32, torch.float64):
    for (R, C) in [(2048, 2048), (4096, 4096), (4096, 8192), (8192, 8192), (8192, 16384)]:
        nb = 2 * R * C * torch.tensor([], dtype=dt).element_size()
        Rn = max(2, -(-3 * L2 // nb))
        ins = [torch.rand((R, C), device="cuda").to(dt) for _ in range(Rn)]
        outs = [torch.empty((C, R), device="cuda", dtype=dt) for _ in range(Rn)]
        fns = [(lambda a=a, o=o: b2.transpose(a, o)) for a, o in zip(ins, outs)]
        res = {}
        for big in (1, 2, 1, 2):
            _lib.tune("transpose.big", big)
            res.setdefault(big, []).append(round(nb / graph_us(fns, max(2 * Rn, 16)) / 1e3))
        _lib.tune("transpose.big", 1)
        assert all(torch.equal(o, a.t()) for a, o in zip(ins, outs))
        print(json.dumps({"dtype": str(dt)[6:], "shape": [R, C], "default": res[1], "big_tiles": res[2]}), flush=True)
        del ins, outs, fns
        torch.cuda.empty_cache()
