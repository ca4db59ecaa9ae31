"""Forward + backward substitution time over a factored SPD matrix, and the
solution (optionally saved, for A/B comparisons between builds).
    python tools/trsv_bench.py --n 32768 --b 512 --reps 10 --save /tmp/x.npy"""
import argparse
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2605_13209_b200 as hs
from paper_2605_13209_b200 import hsolve as H


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=32768)
    ap.add_argument("--b", type=int, default=512)
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--save", default=None)
    a = ap.parse_args()
    rt = hs.Runtime(stream=torch.cuda.current_stream().cuda_stream)
    m = hs.generate_spd_device(rt, a.n, a.b, seed=42)
    L = hs.DeviceMatrix(rt, a.n, a.b)
    L.copy_from(m)
    H.potrf_device(rt, L)
    rhs = torch.from_numpy(hs.generate_rhs(a.n, a.b, 42).values).cuda()
    x = torch.empty_like(rhs)
    ts = []
    for rep in range(a.reps + 1):
        x.copy_(rhs)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        s.record()
        H.trsv_device(rt, L, x.data_ptr(), upper=False)
        H.trsv_device(rt, L, x.data_ptr(), upper=True)
        e.record()
        e.synchronize()
        if rep:
            ts.append(s.elapsed_time(e))
    res = H.true_residual_device(rt, m, x.data_ptr(), rhs.data_ptr())
    rel = res / float(torch.linalg.vector_norm(rhs[:a.n]))
    floor = 2 * (a.n * (a.n + a.b) / 2 * 8) / 7.2e12 * 1e3
    print(f"n={a.n} b={a.b}: "
          f"{statistics.median(ts):.3f} ms (min {min(ts):.3f}; HBM floor ~{floor:.2f} ms), "
          f"rel residual {rel:.3e}", flush=True)
    if a.save:
        np.save(a.save, x.cpu().numpy())


if __name__ == "__main__":
    main()
