"""Read-only HBM bandwidth of this B200 (the CG SYMV roofline), two ways."""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_13209_b200 as hs  # noqa: E402

rt = hs.Runtime()
out = {}
for mode, name in [(0, "bulk_copy_ring_32KB_5stage_148cta"), (1, "ldg128_streaming")]:
    g = C.c_double()
    hs.hsolve._check(rt._L.hs_probe_hbm_read(rt.ctx, 4 << 30, mode, 5, C.byref(g)))
    out[name] = round(g.value, 1)
print(json.dumps(out))
