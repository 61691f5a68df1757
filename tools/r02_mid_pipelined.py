"""Mid-size aligned transposes (the paper's 4096^2 and neighbours) on the pipelined
clock (one CUDA graph of back-to-back launches over rotating inputs >= 3x L2): LDG path
vs every forced cp.async geometry (transpose.cpa = 2, variants 0-11). GB/s, parity-checked."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2605_13864_b200 as b2  # noqa: E402
from paper_2605_13864_b200 import _lib  # noqa: E402

L2 = 126 << 20


def graph_us(fns, K):
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


SET = [("ldg", 0, 0)] + [(f"v{v}", 2, v) for v in range(12)]
for dt, R, C in [(torch.float32, 4096, 4096), (torch.float32, 2048, 8192), (torch.bfloat16, 4096, 8192),
                 (torch.float64, 4096, 2048)]:
    esz = torch.tensor([], dtype=dt).element_size()
    nb = 2 * R * C * esz
    n = max(2, -(-3 * L2 // (R * C * esz)))
    ins = [torch.empty((R, C), device="cuda").uniform_().to(dt) for _ in range(n)]
    outs = [torch.empty((C, R), device="cuda", dtype=dt) for _ in range(n)]
    rec = {"dtype": str(dt).split(".")[-1], "shape": [R, C], "copies": n}
    for rep in range(2):
        for name, cpa, v in SET:
            _lib.tune("transpose.cpa", cpa)
            _lib.tune("transpose.cpa_variant", v)
            us = graph_us([lambda i=i: b2.transpose(ins[i], outs[i]) for i in range(n)], max(2 * n, 16))
            rec.setdefault(name, []).append(round(nb / us / 1e3, 1))
            iv = torch.int16 if esz == 2 else (torch.int32 if esz == 4 else torch.int64)
            assert torch.equal(outs[0].view(iv), ins[0].t().contiguous().view(iv)), (name, R, C)
    _lib.tune("transpose.cpa", 1)
    _lib.tune("transpose.cpa_variant", 0)
    print(json.dumps(rec), flush=True)
    del ins, outs
    torch.cuda.empty_cache()
