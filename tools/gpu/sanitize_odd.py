import os, sys
sys.path.insert(0, os.getcwd())
import torch
import paper_2605_13209_b200 as hs
from paper_2605_13209_b200 import hsolve as H
rt = hs.Runtime(stream=torch.cuda.current_stream().cuda_stream)
# SIMT Cholesky path (b % 128 != 0) + substitutions
n, b = 600, 100
m = hs.generate_spd_device(rt, n, b, seed=42)
orig = hs.generate_spd_device(rt, n, b, seed=42)
rhs = torch.from_numpy(hs.generate_rhs(n, b, 42).values).cuda()
x = torch.zeros_like(rhs)
sp = hs.solve_spd_device(rt, m, rhs.data_ptr(), x.data_ptr(), a_orig=orig)
print("simt chol", sp.true_residual)
# CG: memory-order walk + finalize kernel (b = 512) and the generic SYMV (b = 7)
for n, b in [(2048, 512), (300, 7)]:
    m = hs.generate_spd_device(rt, n, b, seed=42)
    rhs = torch.from_numpy(hs.generate_rhs(n, b, 42).values).cuda()
    x = torch.zeros_like(rhs)
    st = hs.solve_cg_device(rt, m, rhs.data_ptr(), x.data_ptr(), hs.SolverConfig(block_size=b, eps=1e-300, max_iters=8))
    print("cg", n, b, st.iterations)
