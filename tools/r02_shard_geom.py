"""cp.async tile geometries (transpose.cpa = 2, variants 0-9) vs the auto geometry and
the LDG path on the strong-scaling shard shapes (4096 / 8192 x 32768 fp32)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2605_13864_b200 as b2  # noqa: E402
from paper_2605_13864_b200 import _lib  # noqa: E402
from r02_shard_shapes import timeit  # noqa: E402

SET = [("ldg", 0, 0), ("auto", 1, 0)] + [(f"v{v}", 2, v) for v in range(10)]
for R, C in [(4096, 32768), (8192, 32768)]:
    a = torch.empty((R, C), device="cuda").uniform_()
    o = torch.empty((C, R), device="cuda")
    rec = {"shape": [R, C]}
    for rep in range(2):
        for name, cpa, v in SET:
            _lib.tune("transpose.cpa", cpa)
            _lib.tune("transpose.cpa_variant", v)
            rec.setdefault(name, []).append(round(2 * R * C * 4 / timeit(lambda: b2.transpose(a, o)) / 1e6, 1))
    _lib.tune("transpose.cpa", 1)
    _lib.tune("transpose.cpa_variant", 0)
    print(json.dumps(rec), flush=True)
    del a, o
