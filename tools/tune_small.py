"""Reduce latency at mid sizes (2^20..2^26) with L2 flushed: residency / variant sweep."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2605_13864_b200 as b2  # noqa: E402
from paper_2605_13864_b200 import _lib  # noqa: E402

flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
res = []
for k in (20, 22, 24, 26):
    x = torch.rand(1 << k, device="cuda")
    r = torch.empty(1, device="cuda")
    for var, cpss in [(0, [1, 2, 3, 4]), (2, [4, 6, 8]), (3, [1, 2])]:
        for cps in cpss:
            _lib.tune("reduce.variant", var)
            _lib.tune("reduce.ctas_per_sm", cps)
            ts = []
            for i in range(25):
                flush.fill_(float(i))
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                b2.reduce_sum(x, out=r)
                e1.record()
                torch.cuda.synchronize()
                if i >= 5:
                    ts.append(e0.elapsed_time(e1))
            ms = statistics.median(ts)
            res.append({"log2n": k, "variant": var, "cps": cps, "us": ms * 1e3, "GBps": (1 << k) * 4 / ms / 1e6})
            print(json.dumps(res[-1]), flush=True)
_lib.tune("reduce.variant", 0)
_lib.tune("reduce.ctas_per_sm", 0)
json.dump(res, open("gpurun_out/tune_small.json", "w"), indent=1)
