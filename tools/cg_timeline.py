"""SYMV launch timeline inside CG (debug build
tools/libhsolve_cuda_symvtiming.so: `python -m paper_2605_13209_b200._build
--symv-timing`): per launch the first
CTA start / last CTA end (globaltimer), so the gaps between SYMVs (finalize,
vector kernels, launch latency, host stalls) can be seen iteration by
iteration."""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2605_13209_b200 import _lib  # noqa: E402

LIB = os.path.join(ROOT, "tools", "libhsolve_cuda_symvtiming.so")
_lib.lib_path = lambda: LIB
import torch  # noqa: E402

import paper_2605_13209_b200 as hs  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
b = int(sys.argv[2]) if len(sys.argv) > 2 else 128
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 200
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 3
mode = sys.argv[5] if len(sys.argv) > 5 else ""
dbg = C.CDLL(LIB)
dbg.hs_debug_symv_ts.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int]
dbg.hs_debug_fin_ts.argtypes = [C.c_void_p, C.c_int, C.c_int]
dbg.hs_debug_tail_ts.argtypes = [C.c_void_p, C.c_int, C.c_int]
dbg.hs_debug_tail_cta.argtypes = [C.c_void_p]
dbg.hs_debug_symv_fin_end.argtypes = [C.c_void_p, C.c_int, C.c_int]
rt = (hs.Runtime(device=0, stream=torch.cuda.current_stream().cuda_stream)
      if "torchstream" in mode else hs.Runtime())
m = hs.generate_spd_device(rt, n, b, seed=42)
rhs = torch.from_numpy(hs.generate_rhs(n, b, 42).values).cuda()
x = torch.zeros_like(rhs)
from paper_2605_13209_b200 import hsolve as H  # noqa: E402
y = torch.zeros_like(rhs)
dbg.hs_debug_symv_ts(None, 0, 1, 0)
for _ in range(20):
    H.symv_device(rt, m, rhs.data_ptr(), y.data_ptr())
torch.cuda.synchronize()
buf0 = (C.c_ulonglong * (2 * 4096))()
dbg.hs_debug_symv_ts(buf0, 4096, 0, 0)
d0 = sorted((buf0[2 * k + 1] - buf0[2 * k]) / 1e3 for k in range(4096) if buf0[2 * k + 1])
print(f"standalone hs_symv: {len(d0)} launches, SYMV kernel us median {d0[len(d0) // 2]:.1f} "
      f"min {d0[0]:.1f} max {d0[-1]:.1f}")
cfg = hs.SolverConfig(block_size=b, eps=1e-300, max_iters=iters)
hs.solve_cg_device(rt, m, rhs.data_ptr(), x.data_ptr(), cfg)
torch.cuda.synchronize()
for rep in range(reps):
    dbg.hs_debug_symv_ts(None, 0, 1, 0)
    dbg.hs_debug_fin_ts(None, 0, 1)
    dbg.hs_debug_tail_ts(None, 0, 1)
    dbg.hs_debug_symv_fin_end(None, 0, 1)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    hs.solve_cg_device(rt, m, rhs.data_ptr(), x.data_ptr(), cfg)
    e1.record()
    e1.synchronize()
    buf = (C.c_ulonglong * (2 * 4096))()
    dbg.hs_debug_symv_ts(buf, 4096, 0, 0)
    fb = (C.c_ulonglong * (5 * 4096))()
    dbg.hs_debug_fin_ts(fb, 4096, 0)
    fin = sorted(tuple(fb[5 * k + i] for i in range(5)) for k in range(4096)
                 if fb[5 * k + 2] != 0)
    ts = [(buf[2 * k], buf[2 * k + 1]) for k in range(4096) if buf[2 * k + 1] != 0]
    ts.sort()
    dur = [(e - s) / 1e3 for s, e in ts]
    gaps = [(ts[k][0] - ts[k - 1][1]) / 1e3 for k in range(1, len(ts))]
    sd, sg = sorted(dur), sorted(gaps)
    print(f"rep {rep}: {e0.elapsed_time(e1) / iters:.3f} ms/iter; {len(ts)} SYMV launches; "
          f"duration us median {sd[len(sd) // 2]:.1f} max {sd[-1]:.1f}; "
          f"gap us median {sg[len(sg) // 2]:.1f} p90 {sg[9 * len(sg) // 10]:.1f} "
          f"max {sg[-1]:.1f}; total gap {sum(gaps) / 1e3:.2f} ms")
    # per iteration: SYMV end -> finalize start, finalize sums, dot epilogue,
    # finalize end -> next SYMV start (the two vector kernels + launch gaps)
    br = []
    for k in range(len(ts) - 1):
        s_end, nxt = ts[k][1], ts[k + 1][0]
        f = [x for x in fin if s_end <= x[0] < nxt]
        if f:
            f0, f1, f2, f3, f4 = f[0]
            br.append(((f0 - s_end) / 1e3, (f1 - f0) / 1e3, (f2 - f1) / 1e3, (nxt - f2) / 1e3,
                       (f3 - f0) / 1e3, f4 / 1e3))
    if br:
        med = [sorted(x[i] for x in br)[len(br) // 2] for i in range(6)]
        print("   gap breakdown us (median): SYMV end->finalize start %.1f, sums %.1f, "
              "dot epilogue %.1f, finalize end->next SYMV %.1f; CTA start spread %.1f, "
              "longest CTA sums %.1f" % tuple(med))
    fe = (C.c_ulonglong * 4096)()
    dbg.hs_debug_symv_fin_end(fe, 4096, 0)
    fends = sorted(v for v in fe if v)
    fin_tail = []
    for s0, s1 in ts:
        f = [v for v in fends if s1 - 100000 <= v < s1 + 200000]
        if f:
            fin_tail.append((f[0] - s1) / 1e3)
    if fin_tail:
        fin_tail.sort()
        print("   in-kernel finalize: last finalize warp end - streaming end us: median %.1f "
              "p90 %.1f max %.1f" % (fin_tail[len(fin_tail) // 2],
                                     fin_tail[9 * len(fin_tail) // 10], fin_tail[-1]))
    tb = (C.c_ulonglong * (7 * 4096))()
    dbg.hs_debug_tail_ts(tb, 4096, 0)
    tail = sorted(tuple(tb[7 * k + i] for i in range(7)) for k in range(4096)
                  if tb[7 * k + 5] != 0)
    tr = []
    for k in range(len(ts) - 1):
        s_end, nxt = ts[k][1], ts[k + 1][0]
        f = [x for x in tail if s_end <= x[0] < nxt]
        if f:
            t0, t1, t2, t3, t4, t5, t6 = f[0]
            tr.append(((t0 - s_end) / 1e3, (t1 - t0) / 1e3, (t2 - t1) / 1e3, (t6 - t1) / 1e3,
                       (t3 - t2) / 1e3, (t4 - t3) / 1e3, (t5 - t4) / 1e3, (nxt - t5) / 1e3))
    if tr:
        med = [sorted(x[i] for x in tr)[len(tr) // 2] for i in range(8)]
        print("   fused tail us (median): SYMV end->tail start %.1f, phase 1 %.1f, "
              "barrier 1 (last arrival->last exit %.1f, ->first exit %.1f), phase 2 %.1f, "
              "barrier 2 %.1f, phase 3 %.1f, tail end->next SYMV %.1f" % tuple(med))
    if tr and rep == 0:
        cb = (C.c_ulonglong * (5 * 1024))()
        dbg.hs_debug_tail_cta(cb)
        rows = [[cb[5 * k + i] for i in range(5)] for k in range(1024) if cb[5 * k + 4]]
        if rows:
            t0 = min(r[0] for r in rows)
            def q(v):
                v = sorted(v)
                return "min %.1f med %.1f p90 %.1f max %.1f" % (v[0], v[len(v) // 2],
                                                               v[9 * len(v) // 10], v[-1])
            print("   per-CTA (us) start offset:", q([(r[0] - t0) / 1e3 for r in rows]))
            print("   per-CTA phase 1 (own start->own end):", q([(r[1] - r[0]) / 1e3 for r in rows]))
            print("   per-CTA phase 1 end offset:", q([(r[1] - t0) / 1e3 for r in rows]))
            print("   per-CTA phase 2:", q([(r[3] - r[2]) / 1e3 for r in rows]))
    big = [(k, round(g, 1)) for k, g in enumerate(gaps) if g > 200]
    if big:
        print("   gaps > 200 us (launch index, us):", big[:20])
    slow = [(k, round(d, 1)) for k, d in enumerate(dur) if d > 1.5 * sd[len(sd) // 2]]
    if slow:
        print("   slow SYMVs (index, us):", slow[:20])
