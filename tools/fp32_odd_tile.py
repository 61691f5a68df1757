import json, os, statistics, sys
sys.path.insert(0, '/root/repo')
import torch
import paper_2605_13864_b200 as b2
from paper_2605_13864_b200 import _lib
def timeit(fn, reps=15):
    for _ in range(3): fn()
    ts=[]
    for _ in range(reps):
        e0,e1=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)
for R,C in [(16385,16383),(4097,8191)]:
    a=torch.rand((R,C),device="cuda"); o=torch.empty((C,R),device="cuda"); nb=2*a.numel()*4
    for rep in range(2):
        for tile,cps in [(0,0),(128,0),(128,1),(128,2),(128,3)]:
            _lib.tune("transpose.scalar_tile",tile); _lib.tune("transpose.scalar_ctas",cps)
            ms=timeit(lambda: b2.transpose(a,o))
            print(json.dumps({"shape":[R,C],"tile":tile or 64,"cps":cps,"GBps":round(nb/ms/1e6),"ok":bool(torch.equal(o,a.t()))}))
