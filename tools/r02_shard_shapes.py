"""Transpose of the strong-scaling shard shapes of the bench (C4 32768^2 split over
N = 2 / 4 / 8 GPUs: 16384 / 8192 / 4096 x 32768 fp32 row blocks): LDG path vs the
cp.async path with several tile-walk band heights (transpose.group; 0 = auto).
Interleaved A B A B, CUDA-event median of 10 launches, inputs > L2; parity-checked."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2605_13864_b200 as b2  # noqa: E402
from paper_2605_13864_b200 import _lib  # noqa: E402


def timeit(fn, reps=10):
    for _ in range(3):
        fn()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)


SETTINGS = [("ldg", {"transpose.cpa": 0}), ("cpa", {})] + \
    [(f"cpa_g{g}", {"transpose.group": g}) for g in (1, 2, 4, 8, 16, 1 << 20)]


def apply(knobs):
    _lib.tune("transpose.cpa", 1)
    _lib.tune("transpose.group", 0)
    for k, v in knobs.items():
        _lib.tune(k, v)


def main():
    for R, C in [(4096, 32768), (8192, 32768), (16384, 32768), (32768, 32768)]:
        a = torch.empty((R, C), device="cuda").uniform_()
        o = torch.empty((C, R), device="cuda")
        rec = {"shape": [R, C]}
        for rep in range(2):
            for name, knobs in SETTINGS:
                apply(knobs)
                ms = timeit(lambda: b2.transpose(a, o))
                rec.setdefault(name, []).append(round(2 * R * C * 4 / ms / 1e6, 1))
        for name, knobs in SETTINGS:
            apply(knobs)
            o.zero_()
            b2.transpose(a, o)
            rec[name + "_ok"] = bool(torch.equal(o, a.t()))
        apply({})
        print(json.dumps(rec), flush=True)
        del a, o
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
