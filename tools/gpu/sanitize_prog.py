# small progressive-SYMV CG solves for compute-sanitizer (memcheck / racecheck / synccheck)
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_2605_13209_b200 as hs
from oracle import Oracle
o = Oracle()
rt = hs.Runtime()
for n, b in [(2048, 128), (1000, 64)]:
    a = o.generate_spd(n, b, seed=3); rhs = o.generate_rhs(n, b, seed=3)
    ref = o.solve_cg(n, b, a, rhs, eps=1e-6)
    r = hs.solve_cg(hs.BlockedSPDMatrix(n, b, a), hs.BlockVector(n, b, rhs),
                    hs.SolverConfig(block_size=b, eps=1e-6, recompute_interval=5), rt)
    x = r.x.values[:n]
    err = np.linalg.norm(x - ref["x"][:n]) / np.linalg.norm(ref["x"][:n])
    print(n, b, r.stats.iterations, ref["iterations"], err, flush=True)
    assert err < 1e-6
print("OK")
