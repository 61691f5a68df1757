"""Odd-pitch (scalar padded-tile path) transposes, GB/s for the current B2K_LIB /
B2K_TUNE: bf16 / fp32 / fp64 over large, mid and small odd shapes. Large shapes
timed with CUDA events (inputs > L2), smaller ones as a CUDA graph over rotating
copies (>= 3x L2). Parity against torch's own transpose on every shape."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2605_13864_b200 as b2  # noqa: E402

L2 = 126 * 1024 * 1024


def graph_time(fns, K):
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
    return statistics.median(ts)


out = {"lib": os.environ.get("B2K_LIB", "in-tree"), "tune": os.environ.get("B2K_TUNE", "")}
for dtn in ("bfloat16", "float32", "float64"):
    dt = getattr(torch, dtn)
    for (H, W) in [(16385, 16383), (8193, 16385), (4097, 8191), (1023, 1025), (2049, 3071)]:
        nb = 2 * H * W * torch.tensor([], dtype=dt).element_size()
        R = max(1, min(32, -(-3 * L2 // nb)))
        ins = [torch.empty((H, W), device="cuda", dtype=dt).uniform_() for _ in range(R)]
        outs = [torch.empty((W, H), device="cuda", dtype=dt) for _ in range(R)]
        fns = [(lambda a=a, o=o: b2.transpose(a, o)) for a, o in zip(ins, outs)]
        ms = graph_time(fns, max(2 * R, 8))
        ok = all(torch.equal(o, a.t()) for a, o in zip(ins, outs))
        out[f"{dtn} {H}x{W}"] = round(nb / ms / 1e6)
        assert ok, (dtn, H, W)
        del ins, outs, fns
        torch.cuda.empty_cache()
print(json.dumps(out), flush=True)
