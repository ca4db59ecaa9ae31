# world-1 NCCL (2D block-cyclic 1x1) factor vs the single-GPU factor
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2605_13209_b200 as hs
from paper_2605_13209_b200 import hsolve as H
rt1 = hs.Runtime()
rtd = hs.Runtime.distributed(0, 0, 1, hs.Runtime.nccl_unique_id())
for n, b in [(8192, 512), (16384, 512), (32768, 512)]:
    m = hs.generate_spd_device(rt1, n, b, seed=42)
    w = hs.DeviceMatrix(rt1, n, b); w.copy_from(m)
    H.potrf_device(rt1, w)
    L1 = w.download(); w.free(); m.free()
    res = []
    for rep in range(2):
        md = hs.generate_spd_device(rtd, n, b, seed=42, cyclic=True)
        try:
            H.potrf_device(rtd, md)
            Ld = md.download()
            res.append(float(np.max(np.abs(Ld - L1))))
        except Exception as e:
            res.append(repr(e)[:80])
        md.free()
    print(os.environ.get("HS_GEMM64"), n, b, res, flush=True)
