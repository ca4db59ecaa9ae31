"""Cholesky factorization time with the trailing update on FP64 DMMA
(slices 0) or emulated FP64 on the INT8 tensor cores (slices 1..8):
    python tools/chol_bench.py --n 32768 --b 512 --slices 0 8
Reports GFLOP/s (n^3/3 / factor time, CUDA events) and the factor's distance
to the DMMA factor."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

if os.environ.get("HS_LIB"):  # A/B against another build of the CUDA library
    from paper_2605_13209_b200 import _lib  # noqa: E402
    _lib.lib_path = lambda: os.environ["HS_LIB"]
import paper_2605_13209_b200 as hs  # noqa: E402
from paper_2605_13209_b200 import hsolve as H  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=32768)
    ap.add_argument("--b", type=int, default=512)
    ap.add_argument("--slices", type=int, nargs="+", default=[0, 8])
    ap.add_argument("--reps", type=int, default=2)
    a = ap.parse_args()
    rt = hs.Runtime(stream=torch.cuda.current_stream().cuda_stream)
    m = hs.generate_spd_device(rt, a.n, a.b, seed=42)
    work = hs.DeviceMatrix(rt, a.n, a.b)
    ref = None
    for s in a.slices:
        rt.set_cholesky_gemm(s)
        best = 1e30
        for _ in range(1 + a.reps):
            work.copy_from(m)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            H.potrf_device(rt, work)
            e1.record()
            e1.synchronize()
            best = min(best, e0.elapsed_time(e1))
        L = torch.from_numpy(work.download()).cuda()
        if ref is None:
            ref = L
            d = 0.0
        else:
            d = float((L - ref).abs().max() / ref.abs().max())
        print(f"n={a.n} b={a.b} slices={s}: {best:.1f} ms = "
              f"{a.n ** 3 / 3 / best / 1e9:.1f} TF/s; max|L-L_dmma|/max|L| = {d:.2e}",
              flush=True)
    rt.close()


if __name__ == "__main__":
    main()
