import sys, os, statistics
sys.path.insert(0, os.getcwd())
import torch
import paper_2605_13864_b200 as b2
for dt, (R, C) in [(torch.bfloat16, (8192, 16384)), (torch.float32, (8192, 16384)), (torch.float32, (32768, 32768))]:
    a = torch.empty((R, C), device="cuda", dtype=dt).uniform_()
    o = torch.empty((C, R), device="cuda", dtype=dt)
    nb = 2 * a.numel() * a.element_size()
    for _ in range(5): b2.transpose(a, o)
    ts = []
    for i in range(200):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); b2.transpose(a, o); e1.record(); torch.cuda.synchronize()
        ts.append(nb / e0.elapsed_time(e1) / 1e6)
    ts.sort()
    print(dt, R, C, [round(ts[int(q * 199)]) for q in (0, .1, .25, .5, .75, .9, 1)])
    print("  seq:", [round(x) for x in ts[:0]])
    # sequence pattern
    ts2 = []
    for i in range(40):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); b2.transpose(a, o); e1.record(); torch.cuda.synchronize()
        ts2.append(round(nb / e0.elapsed_time(e1) / 1e6))
    print("  seq:", ts2)
    del a, o
