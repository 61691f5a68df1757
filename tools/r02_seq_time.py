"""Time of the reference-order fp32 sum (one warp) on C2's 2^24 cells, device entry,
CUDA events; and its bits against the reference's pinned C2 result."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2605_13864_b200 as b2  # noqa: E402

with open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden",
                       "fullsize_ref.json")) as f:
    pin = json.load(f)["C2"][0]
x = torch.from_numpy(np.random.default_rng(pin["seed"]).uniform(pin["lo"], 1, pin["n"]).astype(np.float32)).cuda()
out = torch.zeros(1, device="cuda")
b2.reduce_sum_sequential(x, out=out)
torch.cuda.synchronize()
ts = []
for _ in range(5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    b2.reduce_sum_sequential(x, out=out)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
bits = int(np.float32(out.item()).view(np.uint32))
print(json.dumps({"n": pin["n"], "ms": sorted(ts)[2], "ns_per_cell": sorted(ts)[2] * 1e6 / pin["n"],
                  "bits": bits, "reference_bits": pin["result_f32_bits"], "bit_exact": bits == pin["result_f32_bits"],
                  "reference_seconds_here": pin["ref_seconds"]}))
