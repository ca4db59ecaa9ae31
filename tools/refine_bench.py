"""Mixed-precision SPD solve (hs_solve_spd_refine) against the FP64 DMMA
solve_spd: factor time, refinement steps, final relative residual.
    python tools/refine_bench.py --n 32768 --b 512 --slices 0 4 5 6 8"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2605_13209_b200 as hs
from paper_2605_13209_b200 import hsolve as H


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=32768)
    ap.add_argument("--b", type=int, default=512)
    ap.add_argument("--slices", type=int, nargs="+", default=[0, 4, 5, 6, 8])
    ap.add_argument("--tol", type=float, default=0.0)
    ap.add_argument("--reps", type=int, default=2)
    a = ap.parse_args()
    rt = hs.Runtime(stream=torch.cuda.current_stream().cuda_stream)
    m = hs.generate_spd_device(rt, a.n, a.b, seed=42)
    work = hs.DeviceMatrix(rt, a.n, a.b)
    rhs = torch.from_numpy(hs.generate_rhs(a.n, a.b, 42).values).cuda()
    x = torch.empty_like(rhs)
    # FP64 reference point: copy + factor + substitutions, no refinement
    for rep in range(a.reps):
        work.copy_from(m)
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        H.solve_spd_device(rt, work, rhs.data_ptr(), x.data_ptr())
        e.record()
        e.synchronize()
    res = H.true_residual_device(rt, m, x.data_ptr(), rhs.data_ptr())
    print(f"solve_spd (FP64 DMMA): {s.elapsed_time(e):.1f} ms, rel residual "
          f"{res / float(torch.linalg.vector_norm(rhs)):.2e}", flush=True)
    for sl in a.slices:
        for rep in range(a.reps):
            torch.cuda.synchronize()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            try:
                st = H.solve_spd_refine_device(rt, m, work, rhs.data_ptr(), x.data_ptr(),
                                               slices=sl, max_iters=30, tol=a.tol)
            except hs.HsolveError as ex:
                print(f"slices={sl}: {type(ex).__name__}: {ex}", flush=True)
                break
            e.record()
            e.synchronize()
        else:
            print(f"slices={sl}: total {s.elapsed_time(e):.1f} ms (factor+copy {st.factor_ms:.1f}, "
                  f"solve+refine {st.solve_ms:.1f}), {st.iterations} refinement steps, "
                  f"rel residual {st.rel_residual:.2e}", flush=True)


if __name__ == "__main__":
    main()
