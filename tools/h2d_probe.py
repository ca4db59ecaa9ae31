import sys, time, ctypes as C
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import paper_2605_13209_b200 as hs
from paper_2605_13209_b200 import hsolve as H
from paper_2605_13209_b200._lib import CgStats
n, b = 32768, 128
rt = hs.Runtime()
m = hs.generate_spd_device(rt, n, b, seed=42)
N = n // b; T = N * (N + 1) // 2
host_pg = np.empty(T * b * b); m.download(host_pg)
host_pin = torch.empty(T * b * b, dtype=torch.float64, pin_memory=True); host_pin.numpy()[:] = host_pg
rhs = hs.generate_rhs(n, b, 42).values.copy(); x = np.zeros_like(rhs)
cfg = hs.SolverConfig(block_size=b, eps=1e-300, max_iters=50); p = H._cg_params(cfg)
for name, ptr in (("pageable", host_pg.ctypes.data), ("pinned", host_pin.data_ptr())):
    for rep in range(3):
        st = CgStats()
        t0 = time.perf_counter()
        H._check(rt._L.hs_solve_cg_host(rt.ctx, n, b, C.c_void_p(ptr), C.c_void_p(rhs.ctypes.data), C.byref(p), C.c_void_p(x.ctypes.data), C.byref(st), None))
        t = time.perf_counter() - t0
        print(name, f"call {t*1e3:.1f} ms transfer {st.transfer_ms:.1f} ms -> {T*b*b*8/1e9/(st.transfer_ms*1e-3):.1f} GB/s")
