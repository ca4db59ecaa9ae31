"""Timing of the emulated-FP64 INT8 GEMM (hs_oz_gemm_tiles) against the DMMA
path (hs_gemm_update_tiles) on `count` b x b tile triples:
    python tools/oz_bench.py --b 512 --count 64 [--slices 8]
Wall time per call via CUDA events (the oz call includes slicing and its
scratch allocation); run under ncu for per-kernel times."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2605_13209_b200 as hs  # noqa: E402
from paper_2605_13209_b200 import hsolve as H  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--b", type=int, default=512)
    ap.add_argument("--count", type=int, default=64)
    ap.add_argument("--slices", type=int, default=8)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--phases", action="store_true",
                    help="per-tile phase breakdown from in-kernel timestamps")
    a = ap.parse_args()
    rt = hs.Runtime(stream=torch.cuda.current_stream().cuda_stream)
    b, n = a.b, a.count
    g = torch.Generator(device="cuda").manual_seed(1)
    P = torch.randn(n, b, b, dtype=torch.float64, device="cuda", generator=g)
    Q = torch.randn(n, b, b, dtype=torch.float64, device="cuda", generator=g)
    C = torch.randn(n, b, b, dtype=torch.float64, device="cuda", generator=g)
    flops = 2.0 * n * b ** 3

    def t(fn):
        fn()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        best = 1e30
        for _ in range(a.reps):
            s.record()
            fn()
            e.record()
            e.synchronize()
            best = min(best, s.elapsed_time(e))
        return best

    ms_oz = t(lambda: H._check(rt._L.hs_oz_gemm_tiles(rt.ctx, C.data_ptr(), P.data_ptr(),
                                                      Q.data_ptr(), b, n, a.slices, 0)))
    ms_dm = t(lambda: H.gemm_update_tiles_device(rt, C.data_ptr(), P.data_ptr(), Q.data_ptr(),
                                                 b, n))
    if a.phases:
        import numpy as np
        buf = torch.zeros(148 * 64 * 8, dtype=torch.int64, device="cuda")
        rt._L.hs_oz_set_profile(buf.data_ptr())
        H._check(rt._L.hs_oz_gemm_tiles(rt.ctx, C.data_ptr(), P.data_ptr(), Q.data_ptr(), b, n,
                                        a.slices, 0))
        rt._L.hs_oz_set_profile(None)
        t = buf.view(148, 64, 8).cpu().numpy().astype(np.float64)
        ok = (t[:, 1:-1, :7] > 0).all(axis=2)
        d = lambda x, y: np.median((t[:, 1:-1, y] - t[:, 1:-1, x])[ok])
        per = np.diff(t[:, :, 1], axis=1)
        pmask = (t[:, 1:, 1] > 0) & (t[:, :-1, 1] > 0)
        print(f"per tile (median, ns): tempty wait {d(0, 1):.0f}, MMA issue->commit "
              f"{d(1, 2):.0f}, epi wait tfull {d(3, 4):.0f}, drain {d(4, 5):.0f}, "
              f"barrier {d(5, 7):.0f}, fp64+stage {d(7, 6):.0f}; tile period {np.median(per[pmask]):.0f}")
    print(f"b={b} count={n} slices={a.slices}: oz {ms_oz:.3f} ms = {flops / ms_oz / 1e9:.1f} "
          f"TF/s (FP64-equivalent, incl. slicing+alloc); dmma {ms_dm:.3f} ms = "
          f"{flops / ms_dm / 1e9:.1f} TF/s")
    rt.close()


if __name__ == "__main__":
    main()
