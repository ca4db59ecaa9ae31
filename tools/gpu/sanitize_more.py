import os, sys
sys.path.insert(0, os.getcwd())
import torch
import paper_2605_13209_b200 as hs
from paper_2605_13209_b200 import hsolve as H
which = sys.argv[1]
if which == "cg":
    rt = hs.Runtime(stream=torch.cuda.current_stream().cuda_stream)
    n, b = 4096, 128
    m = hs.generate_spd_device(rt, n, b, seed=42)
    rhs = torch.from_numpy(hs.generate_rhs(n, b, 42).values).cuda()
    x = torch.zeros_like(rhs)
    st = hs.solve_cg_device(rt, m, rhs.data_ptr(), x.data_ptr(), hs.SolverConfig(block_size=b, eps=1e-300, max_iters=60))
    print("cg", st.iterations, st.true_residual)
else:
    rt = hs.Runtime.distributed(0, 0, 1, hs.Runtime.nccl_unique_id())
    n, b = 1536, 512
    m = hs.generate_spd_device(rt, n, b, seed=42, cyclic=True)
    orig = hs.generate_spd_device(rt, n, b, seed=42, cyclic=True)
    rhs = torch.from_numpy(hs.generate_rhs(n, b, 42).values).cuda()
    x = torch.zeros_like(rhs)
    sp = hs.solve_spd_device(rt, m, rhs.data_ptr(), x.data_ptr(), a_orig=orig)
    print("dist", sp.true_residual)
