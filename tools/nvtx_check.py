"""NVTX check: ncu --nvtx --nvtx-include "b2_reduce_sum/" python tools/nvtx_check.py captures
only the two reduce_kernel launches (verified on B200)."""
import os, sys
sys.path.insert(0, os.getcwd())
import torch
import paper_2605_13864_b200 as b2
x = torch.ones(1 << 20, device="cuda")
a = torch.ones(512, 512, device="cuda")
b2.transpose(a); b2.reduce_sum(x); b2.transpose(a); b2.reduce_sum(x)
torch.cuda.synchronize()
