"""Generate the golden fixtures from the REAL reference (oracle/_ref, compiled
from /root/reference/proj/src by oracle/Makefile). Run in the dev container:

    make -C oracle ref && python tests/golden/make_golden.py

Fixtures are small; large arrays are stored as SHA-256 digests of their
little-endian bytes (the oracle must reproduce them bitwise).
"""
import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle import Reference  # noqa: E402


def digest(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype="<f8").tobytes()).hexdigest()


def main():
    r = Reference()
    out = {}
    meta = {}
    # assembly + symv on the reference's own test shape (test_block_kernels.cpp:235)
    a45 = r.generate_spd(45, 8, seed=17)
    x45 = r.generate_rhs(45, 8, seed=10)
    out["spd_45_8_s17"] = a45
    out["rhs_45_8_s10"] = x45
    out["symv_45_8"] = r.symv(45, 8, a45, x45)
    out["inputs_100_2_s42"] = r.generate_inputs(100, 2, 42)
    # cfg1: n=1024, b=128, seed 42 (BASELINE.json configs[0])
    n, b = 1024, 128
    a = r.generate_spd(n, b, seed=42)
    rhs = r.generate_rhs(n, b, seed=42)
    meta["cfg1_spd_sha256"] = digest(a)
    out["cfg1_rhs"] = rhs
    cg = r.solve_cg(n, b, a, rhs, eps=1e-6, max_iters=500, recompute_interval=50,
                    fraction=0.0, workers=4)
    out["cfg1_cg_x"] = cg["x"]
    out["cfg1_cg_trace"] = cg["trace"]
    meta["cfg1_cg"] = dict(iterations=cg["iterations"], u0=cg["u0"],
                           true_residual=cg["true_residual"], converged=cg["converged"])
    sp = r.solve_spd(n, b, a, rhs, workers=4)
    out["cfg1_spd_x"] = sp["x"]
    meta["cfg1_L_sha256"] = digest(sp["L"])
    meta["cfg1_spd_true_residual"] = sp["true_residual"]
    # small Cholesky, full factor (test_cholesky_solver.cpp shapes)
    a128 = r.generate_spd(128, 16, seed=5)
    out["chol_128_16_L"] = r.factorize(128, 16, a128)["L"]
    # heterogeneous CG split (fraction 0.5) is bitwise identical to homogeneous
    cgh = r.solve_cg(128, 16, r.generate_spd(128, 16, seed=99), r.generate_rhs(128, 16, 99),
                     eps=1e-9, max_iters=300, fraction=0.5, workers=2)
    out["cg_128_16_s99_x"] = cgh["x"]
    out["cg_128_16_s99_trace"] = cgh["trace"]
    meta["cg_128_16_s99_ledger"] = cgh["ledger"]
    np.savez_compressed(os.path.join(HERE, "reference_golden.npz"), **out)
    with open(os.path.join(HERE, "reference_golden.json"), "w") as f:
        json.dump(meta, f, indent=1, sort_keys=True)
    print("wrote", sorted(out), sorted(meta))


if __name__ == "__main__":
    main()
