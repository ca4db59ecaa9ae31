import sys, os
sys.path.insert(0, os.getcwd())
import torch, numpy as np
import paper_2605_13209_b200 as hs
from paper_2605_13209_b200 import hsolve as H
rt = hs.Runtime(stream=torch.cuda.current_stream().cuda_stream)
for n, b in [(4096, 512), (8192, 512), (16384, 512), (8192, 256), (4096, 128)]:
    m = hs.generate_spd_device(rt, n, b, seed=42)
    Ls = []
    for rep in range(3):
        w = hs.DeviceMatrix(rt, n, b); w.copy_from(m)
        H.potrf_device(rt, w)
        Ls.append(w.download()); w.free()
    d = max(float(np.max(np.abs(Ls[0] - L))) for L in Ls[1:])
    # reconstruction residual via solve
    rhs = torch.from_numpy(hs.generate_rhs(n, b, 42).values).cuda()
    y = torch.empty_like(rhs)
    w = hs.DeviceMatrix(rt, n, b); w.copy_from(m)
    sp = hs.solve_spd_device(rt, w, rhs.data_ptr(), y.data_ptr(), a_orig=m)
    print(os.environ.get("HS_GEMM64"), n, b, "run-to-run max diff", d, "rel residual", sp.true_residual / float(torch.linalg.vector_norm(rhs)), flush=True)
    w.free(); m.free()
