"""Launch the latency-bound BASELINE cases once each (C1 1024^2 fp32 transpose,
C2 2^24 fp32 sum, the paper's 4096^2, plus 2^20 / 2^22 / 2^26 sums and 2048^2) so
ncu's cache-flushed per-kernel durations show the kernels' own cold-L2 time, free
of the ~6 us CUDA-event floor (tools/ncu_small.sh)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2605_13864_b200 as b2  # noqa: E402

for n in [1024, 2048, 4096]:
    a = torch.rand((n, n), device="cuda")
    o = torch.empty_like(a)
    for _ in range(2):
        b2.transpose(a, o)
for logn in [20, 22, 24, 26]:
    x = torch.rand(1 << logn, device="cuda")
    r = torch.empty(1, device="cuda")
    for _ in range(2):
        b2.reduce_sum(x, out=r)
torch.cuda.synchronize()
