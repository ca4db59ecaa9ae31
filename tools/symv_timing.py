"""Per-CTA start / end times of the SYMV (debug build
tools/libhsolve_cuda_symvtiming.so: `python -m paper_2605_13209_b200._build
--symv-timing`; the kernel printf's one line per CTA). Run a few CG iterations and summarise
each launch: spread of CTA start and end times, per-CTA bytes/time."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run_child(n, b, iters):
    sys.path.insert(0, ROOT)
    from paper_2605_13209_b200 import _lib
    _lib.lib_path = lambda: os.path.join(ROOT, "tools", "libhsolve_cuda_symvtiming.so")
    import ctypes as C
    import torch
    import paper_2605_13209_b200 as hs
    rt = hs.Runtime()
    dbg = C.CDLL(_lib.lib_path())
    dbg.hs_debug_symv_ts.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int]
    dbg.hs_debug_symv_ts(None, 0, 1, 1)  # reset, per-CTA printf on
    m = hs.generate_spd_device(rt, n, b, seed=42)
    rhs = torch.from_numpy(hs.generate_rhs(n, b, 42).values).cuda()
    x = torch.zeros_like(rhs)
    hs.solve_cg_device(rt, m, rhs.data_ptr(), x.data_ptr(),
                       hs.SolverConfig(block_size=b, eps=1e-300, max_iters=iters))
    torch.cuda.synchronize()


def main():
    n, b, iters = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
    if len(sys.argv) > 4 and sys.argv[4] == "child":
        run_child(n, b, iters)
        return
    out = subprocess.run([sys.executable, __file__, str(n), str(b), str(iters), "child"],
                         capture_output=True, text=True).stdout
    rows = [ln.split()[1:] for ln in out.splitlines() if ln.startswith("symvts")]
    rows = [(int(c), int(sm), int(sl), int(t0), int(t1)) for c, sm, sl, t0, t1 in rows]
    # group into launches by start time gaps
    rows.sort(key=lambda r: r[3])
    launches, cur = [], [rows[0]]
    for r in rows[1:]:
        if r[3] - cur[-1][3] > 50_000:  # 50 us
            launches.append(cur)
            cur = []
        cur.append(r)
    launches.append(cur)
    for k in range(1, len(launches)):
        gap = min(r[3] for r in launches[k]) - max(r[4] for r in launches[k - 1])
        print(f"gap before launch {k}: {gap / 1e3:.1f} us (end of SYMV -> next SYMV start)")
    for k, L in enumerate(launches):
        t0 = min(r[3] for r in L)
        starts = sorted(r[3] - t0 for r in L)
        ends = sorted(r[4] - t0 for r in L)
        rates = sorted(r[2] * 32768 / (r[4] - r[3]) for r in L)  # GB/s per CTA
        tot = sum(r[2] for r in L) * 32768
        print(f"launch {k}: ctas {len(L)}  start spread {starts[-1] / 1e3:.1f} us  "
              f"end: min {ends[0] / 1e3:.1f} p10 {ends[len(ends) // 10] / 1e3:.1f} "
              f"median {ends[len(ends) // 2] / 1e3:.1f} max {ends[-1] / 1e3:.1f} us  "
              f"per-CTA GB/s min {rates[0]:.1f} med {rates[len(rates) // 2]:.1f} "
              f"max {rates[-1]:.1f}  aggregate {tot / ends[-1]:.0f} GB/s")
        if k == 1:
            slow = sorted(L, key=lambda r: -(r[4] - t0))[:8]
            print("   slowest CTAs (cta, sm, slabs, end us):",
                  [(r[0], r[1], r[2], round((r[4] - t0) / 1e3, 1)) for r in slow])


if __name__ == "__main__":
    main()
