"""bf16 odd-pitch transposes at the defaults (GB/s + parity)."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2605_13864_b200 as b2  # noqa: E402

L2 = 126 * 1024 * 1024
flush = torch.ones(2 * L2 // 4, device="cuda")
for R, C in [(4097, 8191), (16385, 16383), (16385, 32767), (1023, 1025), (33, 65)]:
    a = torch.empty((R, C), device="cuda", dtype=torch.bfloat16).uniform_()
    o = torch.empty((C, R), device="cuda", dtype=torch.bfloat16)
    nb = 2 * a.numel() * 2
    ts = []
    for i in range(18):
        if nb < 4 * L2:
            flush.sum()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        b2.transpose(a, o)
        e1.record()
        torch.cuda.synchronize()
        if i >= 3:
            ts.append(e0.elapsed_time(e1))
    print(json.dumps({"shape": [R, C], "GBps": nb / statistics.median(ts) / 1e6, "ok": bool(torch.equal(o, a.t()))}))
