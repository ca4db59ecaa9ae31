"""Golden fixtures at the BASELINE.json full sizes, generated from the REAL
reference (oracle/_ref, compiled from /root/reference/proj/src by
oracle/Makefile). Run once in the dev container (the Cholesky takes ~12 min
on 8 cores):

    make -C oracle ref && python tests/golden/make_golden_full.py [cg] [chol]

* ``reference_cfg2_cg.npz`` — configs[1]: CG n=32768, b=128, seed 42,
  eps 1e-6 (SolverConfig defaults): x, the (u, alpha, beta) trace,
  iterations, u0, true residual (cg_solver.cpp:223-368).
* ``reference_cfg3_chol.npz`` — configs[2]: solve_spd n=32768, b=512,
  seed 42: x, true residual, and 16 sampled elements of every lower tile
  of L (positions from a seeded generator, stored with the values;
  cholesky_solver.cpp:275-331). The full factor (4.36 GB) is not stored.
"""
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle import Reference  # noqa: E402

SAMPLES_PER_TILE = 16


def l_sample_positions(n: int, b: int, seed: int = 2026) -> np.ndarray:
    """Flat packed offsets of SAMPLES_PER_TILE elements per lower tile (on or
    below the diagonal inside diagonal tiles, logical rows/cols < n)."""
    N = (n + b - 1) // b
    g = np.random.default_rng(seed)
    out = []
    for i in range(N):
        for j in range(i + 1):
            base = (i * (i + 1) // 2 + j) * b * b
            k = 0
            while k < SAMPLES_PER_TILE:
                r, c = int(g.integers(b)), int(g.integers(b))
                if i == j and c > r:
                    r, c = c, r
                if i * b + r >= n or j * b + c >= n:
                    continue
                out.append(base + r * b + c)
                k += 1
    return np.asarray(out, dtype=np.int64)


def make_cg(r: Reference) -> None:
    n, b = 32768, 128
    t0 = time.time()
    a = r.generate_spd(n, b, seed=42)
    rhs = r.generate_rhs(n, b, seed=42)
    cg = r.solve_cg(n, b, a, rhs, eps=1e-6, max_iters=500, recompute_interval=50)
    np.savez_compressed(os.path.join(HERE, "reference_cfg2_cg.npz"),
                        x=cg["x"][:n], trace=cg["trace"],
                        iterations=cg["iterations"], u0=cg["u0"],
                        true_residual=cg["true_residual"], converged=cg["converged"])
    print(f"cfg2 CG: {cg['iterations']} iterations, {time.time() - t0:.1f} s", flush=True)


def make_chol(r: Reference) -> None:
    n, b = 32768, 512
    t0 = time.time()
    a = r.generate_spd(n, b, seed=42)
    rhs = r.generate_rhs(n, b, seed=42)
    sp = r.solve_spd(n, b, a, rhs)
    pos = l_sample_positions(n, b)
    np.savez_compressed(os.path.join(HERE, "reference_cfg3_chol.npz"),
                        x=sp["x"][:n], true_residual=sp["true_residual"],
                        l_pos=pos, l_val=sp["L"][pos], max_abs_a=np.max(np.abs(a)),
                        status=sp["status"])
    print(f"cfg3 Cholesky: status {sp['status']}, {time.time() - t0:.1f} s", flush=True)


if __name__ == "__main__":
    which = set(sys.argv[1:]) or {"cg", "chol"}
    ref = Reference()
    if "cg" in which:
        make_cg(ref)
    if "chol" in which:
        make_chol(ref)
