"""Aligned mid-size transposes (64-256 MB inputs, below the cp.async path's 256-MB
threshold): LDG path vs the cp.async auto geometry with / without the evict-first
hint (transpose.cpa = 2, variants 10 / 11). CUDA-event median of 10 launches over
rotating copies (>= 512 MB in total); parity-checked."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2605_13864_b200 as b2  # noqa: E402
from paper_2605_13864_b200 import _lib  # noqa: E402


def timeit(fn, reps=10):
    import statistics
    for _ in range(3):
        fn(0)
    ts = []
    for i in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn(i)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)


SET = [("ldg", 0, 0), ("cpa_nohint", 2, 10), ("cpa_hint", 2, 11)]
cases = [(torch.float32, 4096, 4096), (torch.float32, 4096, 8192), (torch.float32, 8192, 8192),
         (torch.bfloat16, 8192, 8192), (torch.bfloat16, 8192, 16384), (torch.float64, 4096, 4096),
         (torch.float64, 4096, 8192)]
for dt, R, C in cases:
    esz = torch.tensor([], dtype=dt).element_size()
    ncopy = max(1, min(8, (512 << 20) // (R * C * esz)))
    ins = [torch.empty((R, C), device="cuda").uniform_().to(dt) for _ in range(ncopy)]
    outs = [torch.empty((C, R), device="cuda", dtype=dt) for _ in range(ncopy)]
    rec = {"dtype": str(dt).split(".")[-1], "shape": [R, C], "MB": R * C * esz >> 20}
    for rep in range(2):
        for name, cpa, v in SET:
            _lib.tune("transpose.cpa", cpa)
            _lib.tune("transpose.cpa_variant", v)
            ms = timeit(lambda i: b2.transpose(ins[i % ncopy], outs[i % ncopy]))
            rec.setdefault(name, []).append(round(2 * R * C * esz / ms / 1e6, 1))
    iv = torch.int16 if esz == 2 else (torch.int32 if esz == 4 else torch.int64)
    for name, cpa, v in SET:
        _lib.tune("transpose.cpa", cpa)
        _lib.tune("transpose.cpa_variant", v)
        outs[0].zero_()
        b2.transpose(ins[0], outs[0])
        rec[name + "_ok"] = bool(torch.equal(outs[0].view(iv), ins[0].t().contiguous().view(iv)))
    _lib.tune("transpose.cpa", 1)
    _lib.tune("transpose.cpa_variant", 0)
    print(json.dumps(rec), flush=True)
    del ins, outs
    torch.cuda.empty_cache()
