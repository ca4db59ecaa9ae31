"""Small driver for ncu captures (one GPU): runs a few CG iterations and/or
one Cholesky factorization so `ncu --metrics gpu__time_duration.sum` gives the
per-launch list, and `ncu --set full -k regex:...` the top-kernel report.

    python tools/prof_run.py cg   --n 32768 --b 128 --iters 6
    python tools/prof_run.py chol --n 16384 --b 512
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2605_13209_b200 as hs  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("what", choices=["cg", "chol"])
    ap.add_argument("--n", type=int, default=32768)
    ap.add_argument("--b", type=int, default=128)
    ap.add_argument("--iters", type=int, default=6)
    ap.add_argument("--dist", action="store_true",
                    help="world-1 NCCL context, 2D block-cyclic Cholesky path")
    ap.add_argument("--solve", type=int, default=0,
                    help="after the factorization: this many timed forward + back substitutions")
    ap.add_argument("--slices", type=int, default=0,
                    help="Cholesky trailing update on the INT8 tensor cores (0: DMMA)")
    a = ap.parse_args()
    rt = (hs.Runtime.distributed(0, 0, 1, hs.Runtime.nccl_unique_id()) if a.dist
          else hs.Runtime())
    m = hs.generate_spd_device(rt, a.n, a.b, seed=42, cyclic=a.dist and a.what == "chol")
    if a.what == "cg":
        rhs = torch.from_numpy(hs.generate_rhs(a.n, a.b, 42).values).cuda()
        x = torch.zeros_like(rhs)
        cfg = hs.SolverConfig(block_size=a.b, eps=1e-300, max_iters=a.iters)
        st = hs.solve_cg_device(rt, m, rhs.data_ptr(), x.data_ptr(), cfg)
        print("cg iterations", st.iterations)
    else:
        rt.set_cholesky_gemm(a.slices)
        st = hs.potrf_device(rt, m)
        print("factor ms", st.factor_ms)
        if a.solve:
            v = torch.from_numpy(hs.generate_rhs(a.n, a.b, 42).values).cuda()
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
            for _ in range(a.solve):
                ev[0].record()
                hs.trsv_device(rt, m, v.data_ptr(), False)
                ev[1].record()
                hs.trsv_device(rt, m, v.data_ptr(), True)
                ev[2].record()
                torch.cuda.synchronize()
                print("trsv lower / upper ms %.3f %.3f" % (ev[0].elapsed_time(ev[1]),
                                                          ev[1].elapsed_time(ev[2])))
    torch.cuda.synchronize()
    rt.close()


if __name__ == "__main__":
    main()
