"""cp.async-loaded transpose (transpose.cpa = 1, variants 0-4) vs the default
LDG-staged path on aligned shapes: fp32 C4 32768^2, bf16 / fp64 4-GiB matrices,
ragged and mid sizes. Interleaved A B A B on one box, CUDA-event median of 10
launches (inputs > L2 except the mid sizes, which rotate 8 copies); every
setting is parity-checked against torch's transpose (bit-exact)."""
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


SETTINGS = [("ldg", {"transpose.cpa": 0}), ("auto", {"transpose.cpa": 1}),
            ("auto_nohint", {"transpose.cpa": 1, "transpose.cpa_hint": 0})] + \
    [(f"cpa{v}", {"transpose.cpa": 2, "transpose.cpa_variant": v}) for v in range(10)]
if len(sys.argv) > 1:
    SETTINGS = [s for s in SETTINGS if s[0] in sys.argv[1].split(",")]


def apply(knobs):
    _lib.tune("transpose.cpa", 1)
    _lib.tune("transpose.cpa_variant", 0)
    _lib.tune("transpose.cpa_hint", 1)
    for k, v in knobs.items():
        _lib.tune(k, v)


cases = [(torch.float32, 32768, 32768), (torch.bfloat16, 32768, 65536), (torch.float64, 16384, 32768),
         (torch.float32, 32000, 32008), (torch.float32, 8192, 16384), (torch.float32, 4096, 4096),
         (torch.bfloat16, 8192, 16384)]
for dt, R, C in cases:
    esz = torch.tensor([], dtype=dt).element_size()
    ncopy = max(1, min(8, (512 << 20) // (R * C * esz)))
    ins = [torch.empty((R, C), device="cuda", dtype=torch.float32 if dt != torch.float64 else dt).uniform_().to(dt)
           for _ in range(ncopy)]
    outs = [torch.empty((C, R), device="cuda", dtype=dt) for _ in range(ncopy)]
    nb = 2 * R * C * esz
    rec = {"dtype": str(dt).split(".")[-1], "shape": [R, C], "copies": ncopy}
    for rep in range(2):
        for name, knobs in SETTINGS:
            apply(knobs)
            ms = timeit(lambda i: b2.transpose(ins[i % ncopy], outs[i % ncopy]))
            rec.setdefault(name, []).append(round(nb / ms / 1e6, 1))
    for name, knobs in SETTINGS:
        apply(knobs)
        outs[0].zero_()
        b2.transpose(ins[0], outs[0])
        torch.cuda.synchronize()
        rec[name + "_ok"] = bool(torch.equal(outs[0].view(torch.int16 if esz == 2 else dt),
                                             ins[0].t().contiguous().view(torch.int16 if esz == 2 else dt)))
    apply({})
    print(json.dumps(rec), flush=True)
    del ins, outs
    torch.cuda.empty_cache()
