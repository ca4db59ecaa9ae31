import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_2605_13209_b200 as hs
from oracle import Oracle
o = Oracle(); rt = hs.Runtime()
for n, b, eps, ri in [(4096, 128, 1e-8, 5), (4096, 128, 1e-8, 50), (4096, 128, 1e-6, 5), (2048, 128, 1e-8, 5), (8192, 128, 1e-8, 5)]:
    a = o.generate_spd(n, b, seed=17); rhs = o.generate_rhs(n, b, seed=17)
    ref = o.solve_cg(n, b, a, rhs, eps=eps, recompute_interval=ri)
    r = hs.solve_cg(hs.BlockedSPDMatrix(n, b, a), hs.BlockVector(n, b, rhs),
                    hs.SolverConfig(block_size=b, eps=eps, recompute_interval=ri), rt)
    x = r.x.values[:n]
    e = np.linalg.norm(x - ref["x"][:n]) / np.linalg.norm(ref["x"][:n])
    print(os.environ.get("HS_CG_RECOMP2", "1"), n, b, eps, ri, "gpu", r.stats.iterations, "oracle", ref["iterations"], "x err %.2e" % e, flush=True)
