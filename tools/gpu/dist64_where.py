import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2605_13209_b200 as hs
from paper_2605_13209_b200 import hsolve as H
rt1 = hs.Runtime()
rtd = hs.Runtime.distributed(0, 0, 1, hs.Runtime.nccl_unique_id())
n, b = 16384, 512
N = n // b
m = hs.generate_spd_device(rt1, n, b, seed=42)
H.potrf_device(rt1, m); L1 = m.download(); m.free()
for rep in range(int(os.environ.get("REPS", "3"))):
    md = hs.generate_spd_device(rtd, n, b, seed=42, cyclic=True)
    try:
        H.potrf_device(rtd, md)
    except Exception as e:
        print("rep", rep, repr(e)[:80])
    Ld = md.download(); md.free()
    first = None
    for j in range(N):
        for i in range(j, N):
            t = i * (i + 1) // 2 + j
            A = L1[t*b*b:(t+1)*b*b].reshape(b, b); B = Ld[t*b*b:(t+1)*b*b].reshape(b, b)
            if i == j:
                A = np.tril(A); B = np.tril(B)
            d = np.abs(A - B)
            if d.max() > 0:
                q = [[float(d[r*64:(r+1)*64, c*64:(c+1)*64].max() > 0) for c in range(8)] for r in range(8)]
                first = (i, j, d.max(), q)
                break
        if first: break
    if first:
        i, j, dm, q = first
        print("rep", rep, "first differing tile (i, j) =", (i, j), "max", dm)
        for r in range(8): print("   ", "".join("X" if v else "." for v in q[r]))
    else:
        print("rep", rep, "identical")
