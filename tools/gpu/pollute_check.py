"""Is a factor bitwise stable under unrelated copy traffic? Factors
n=N_ (16384) once clean, then REPS times while a side stream copies
256-MB buffers (torch, independent of the factorization's streams).
DIST_=1: the world-1 distributed (block-cyclic) path."""
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2605_13209_b200 as hs
from paper_2605_13209_b200 import hsolve as H
n, b = int(os.environ.get("N_", "16384")), 512
dist = os.environ.get("DIST_") == "1"
rt = hs.Runtime.distributed(0, 0, 1, hs.Runtime.nccl_unique_id()) if dist else hs.Runtime()


def factor():
    m = hs.generate_spd_device(rt, n, b, seed=42, cyclic=dist)
    err = ""
    try:
        H.potrf_device(rt, m)
    except Exception as e:
        err = repr(e)[:60]
    L = m.download(); m.free()
    return L, err


ref, _ = factor()
a = torch.empty(32 << 20, dtype=torch.float64, device="cuda")
o = torch.empty_like(a)
side = torch.cuda.Stream()
for rep in range(int(os.environ.get("REPS", "4"))):
    with torch.cuda.stream(side):
        for _ in range(300):
            o.copy_(a)
    L, err = factor()
    torch.cuda.synchronize()
    d = np.abs(L - ref)
    print(f"rep {rep} maxdiff {d.max():.3e} ndiff {(d > 0).sum()} {err}", flush=True)
