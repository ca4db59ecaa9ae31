import os, sys
sys.path.insert(0, os.getcwd())
import torch
import paper_2605_13209_b200 as hs
from paper_2605_13209_b200 import hsolve as H
rt = hs.Runtime(stream=torch.cuda.current_stream().cuda_stream)
n, b = 1536, 512
m = hs.generate_spd_device(rt, n, b, seed=42)
w = hs.DeviceMatrix(rt, n, b)
rhs = torch.from_numpy(hs.generate_rhs(n, b, 42).values).cuda()
x = torch.empty_like(rhs)
for sl in (4, 0):
    st = H.solve_spd_refine_device(rt, m, w, rhs.data_ptr(), x.data_ptr(), slices=sl, max_iters=10)
    print(sl, st)
