"""ms per CG iteration (device-resident solve, fixed iteration count) and ms
per standalone SYMV (hs_symv: SYMV + finalize), CUDA events."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

if os.environ.get("HS_LIB"):
    from paper_2605_13209_b200 import _lib  # noqa: E402
    _lib.lib_path = lambda: os.environ["HS_LIB"]
import paper_2605_13209_b200 as hs  # noqa: E402
from paper_2605_13209_b200 import hsolve as H  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
b = int(sys.argv[2]) if len(sys.argv) > 2 else 128
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 200
mode = sys.argv[4] if len(sys.argv) > 4 else ""
rt = (hs.Runtime(device=0, stream=torch.cuda.current_stream().cuda_stream)
      if "torchstream" in mode else hs.Runtime())
if "prof" in mode:
    rt.prof_enable(8)
m = hs.generate_spd_device(rt, n, b, seed=42)
rhs = torch.from_numpy(hs.generate_rhs(n, b, 42).values).cuda()
x = torch.zeros_like(rhs)
y = torch.zeros_like(rhs)
for _ in range(3):
    H.symv_device(rt, m, rhs.data_ptr(), y.data_ptr())
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    H.symv_device(rt, m, rhs.data_ptr(), y.data_ptr())
e1.record()
e1.synchronize()
print(f"hs_symv: {e0.elapsed_time(e1) / 20:.3f} ms per call (incl. host sync)")
cfg = hs.SolverConfig(block_size=b, eps=1e-300, max_iters=iters)
hs.solve_cg_device(rt, m, rhs.data_ptr(), x.data_ptr(), cfg)
torch.cuda.synchronize()
import time  # noqa: E402
ts, ws, cs = [], [], []
for rep in range(5):
    torch.cuda.synchronize()
    w0 = time.perf_counter()
    e0.record()
    w1 = time.perf_counter()
    st = hs.solve_cg_device(rt, m, rhs.data_ptr(), x.data_ptr(), cfg)
    w2 = time.perf_counter()
    print(f"  python: call {w1 * 1e3:.3f} -> {w2 * 1e3:.3f} ms monotonic", file=sys.stderr)
    e1.record()
    e1.synchronize()
    w3 = time.perf_counter()
    ts.append(e0.elapsed_time(e1) / iters)
    ws.append(f"{(w1 - w0) * 1e3:.1f}/{(w2 - w1) * 1e3:.1f}/{(w3 - w2) * 1e3:.1f}")
    cs.append(st.wall_ms / iters)
print("cg ms/iteration (events):", " ".join(f"{t:.3f}" for t in ts))
print("cg ms/iteration (library wall_ms):", " ".join(f"{t:.3f}" for t in cs))
print("host ms record/call/sync:", " ".join(ws))
st = hs.solve_cg_device(rt, m, rhs.data_ptr(), x.data_ptr(),
                        hs.SolverConfig(block_size=b, eps=1e-6, max_iters=500))
print(f"converging solve: {st.iterations} iterations, converged {st.converged}, "
      f"true residual / sqrt(u0) = {st.true_residual / st.u0 ** 0.5:.3e}")
