"""One launch of every hot kernel at a bandwidth-relevant size (for an ncu
launch list with DRAM bytes): fp32 / fp64 / bf16 vector transposes, odd-pitch
scalar transposes, int32 / fp32 / int64 reductions, the A.5 family trees."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2605_13864_b200 as b2  # noqa: E402

cases = [(torch.float32, (32768, 32768)), (torch.float64, (16384, 32768)), (torch.bfloat16, (32768, 65536)),
         (torch.float32, (16385, 16383)), (torch.bfloat16, (16385, 16383)), (torch.float64, (8193, 16383))]
for dt, (R, C) in cases:
    a = torch.empty((R, C), device="cuda", dtype=dt).uniform_()
    b2.transpose(a)
    torch.cuda.synchronize()
    del a
    torch.cuda.empty_cache()
n = 1 << 30
for x in (torch.randint(-2**31, 2**31, (n,), device="cuda", dtype=torch.int64).to(torch.int32),
          torch.rand(n, device="cuda"), torch.randint(-2**62, 2**62, (n // 2,), device="cuda", dtype=torch.int64)):
    b2.reduce_sum(x)
    torch.cuda.synchronize()
    del x
xf = torch.rand(n, device="cuda")
for B in (64, 512, 2048):
    b2.reduce_tree_partials(xf, B)
torch.cuda.synchronize()
