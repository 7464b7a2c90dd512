import os, sys
sys.path.insert(0, os.getcwd())
import torch
from paper_1107_4958_b200 import _native as nat, filtering, table_kernel
def timed(x, kern, out, iters=7):
    ts=[]
    for i in range(iters+2):
        a,b=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
        a.record(); filtering.separable_filter_batch(x,kern,value_bound=None if x.dtype==torch.uint8 else 255.0,out=out,check=False); b.record(); torch.cuda.synchronize()
        if i>=2: ts.append(a.elapsed_time(b))
    return sorted(ts)[len(ts)//2]
g=torch.Generator(device="cuda").manual_seed(1)
for shape,k,sigma in (((64,1000,1000),3,10.0),((64,1024,1024),3,10.0),((1,4001,4001),4,8.0),((1,4096,4096),4,8.0),((16,1001,1003),3,5.0)):
    kern=table_kernel(k,sigma)
    base=torch.rand(shape,device="cuda",generator=g)*255
    out=torch.empty(shape,device="cuda",dtype=torch.float32)
    res=[]
    for dt in (torch.uint8, torch.float32, torch.float64):
        x=base.to(dt)
        r=[]
        for pol in (0,2):
            with nat.path_policy(pol): r.append(timed(x,kern,out))
        res.append(f"{str(dt).split('.')[-1]}: auto {r[0]:.4f} unfused {r[1]:.4f}")
    print(shape, kern.max_radius, "  ".join(res), flush=True)
