"""Measure the CG iteration-count / solution envelope of the REFERENCE at
n=32768 under changes of rounding order only (TEST INFRASTRUCTURE; dev
container, needs oracle/_ref).

Variants, all on the same seed-42 GP system and rhs (genmat.cpp:114-162):
  * the compiled reference (oracle/_ref) at b = 64, 128, 256: the block size
    changes only the accumulation order of symv_row / row_dot
    (block_kernels.cpp:59-116), not the system;
  * the C restatement compiled with FMA contraction (-mfma
    -ffp-contract=fast) at b = 128: the SYMV's mul-then-add becomes a fused
    multiply-add, the rounding the GPU kernels use;
  * the C restatement with "tile partials" (hso_set_symv_order(1)): every
    tile's contribution to a row summed from 0, then added in ascending j
    (the GPU SYMV's accumulation class);
  * numpy on the dense matrix: one BLAS dgemv per matvec, and a tile-blocked
    matvec (BLAS 128-column panels added in ascending j). Same CG recurrence
    (cg_solver.cpp:252-340) with plain dots.

Prints one JSON object: iterations, u0, true residual, and the relative
distance of each x from the b=128 reference x. The numbers are what
DESIGN.md §4 and tests/test_gpu_fullsize.py quote as the measured envelope.

    python tools/cg_envelope.py [--n 32768] [--out profiles/r02_cg_envelope.json]
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import Oracle, Reference  # noqa: E402


def fma_oracle() -> Oracle:
    so = "/tmp/liboracle_fma.so"
    subprocess.run(["gcc", "-std=c11", "-O3", "-mfma", "-ffp-contract=fast", "-fPIC",
                    "-shared", "-o", so, os.path.join(ROOT, "oracle", "hs_oracle.c"),
                    "-lm", "-lpthread"], check=True)
    return Oracle(so)


def dense_variants(a, rhs, n, b, res, xs):
    N = n // b
    A = np.zeros((n, n))
    for i in range(N):
        for j in range(i + 1):
            k = (i * (i + 1) // 2 + j) * b * b
            t = a[k:k + b * b].reshape(b, b)
            if i == j:
                t = np.tril(t) + np.tril(t, -1).T
            A[i * b:(i + 1) * b, j * b:(j + 1) * b] = t
            if i != j:
                A[j * b:(j + 1) * b, i * b:(i + 1) * b] = t.T
    r0 = rhs[:n].copy()

    def cg(mv, eps=1e-6):
        x = np.zeros(n)
        r = r0.copy()
        s = r.copy()
        u = u0 = r @ r
        for it in range(1, 501):
            t = mv(s)
            al = u / (s @ t)
            x += al * s
            r -= al * t
            un = r @ r
            s = r + (un / u) * s
            u = un
            if u <= eps * eps * u0:
                break
        return it, x, float(np.linalg.norm(r0 - A @ x)), u0

    def tiles(v):
        acc = np.zeros((N, b))
        V = v.reshape(N, b)
        for j in range(N):
            acc += (A[:, j * b:(j + 1) * b] @ V[j]).reshape(N, b)
        return acc.reshape(-1)

    for name, mv in (("numpy dense dgemv", lambda v: A @ v),
                     ("numpy tile-blocked (BLAS 128-column panels)", tiles)):
        t0 = time.time()
        it, x, tr, u0 = cg(mv)
        xs[name] = x
        res["runs"].append(dict(variant=name, iterations=it, u0=float(u0), true_residual=tr,
                                rel_res=tr / np.sqrt(u0), seconds=time.time() - t0))
        print(res["runs"][-1], flush=True)
    del A


def unpad(v, n):
    return np.asarray(v[:n])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=32768)
    ap.add_argument("--blocks", default="64,128,256")
    ap.add_argument("--out", default="")
    args = ap.parse_args()
    n = args.n
    r = Reference()
    res = {"n": n, "eps": 1e-6, "seed": 42, "threads": os.cpu_count(), "runs": []}
    xs = {}
    for b in [int(v) for v in args.blocks.split(",")]:
        t0 = time.time()
        a = r.generate_spd(n, b, seed=42)
        rhs = r.generate_rhs(n, b, seed=42)
        cg = r.solve_cg(n, b, a, rhs, eps=1e-6, max_iters=500, recompute_interval=50)
        xs[f"ref_b{b}"] = unpad(cg["x"], n)
        res["runs"].append(dict(variant=f"reference b={b}", iterations=cg["iterations"],
                                u0=cg["u0"], true_residual=cg["true_residual"],
                                rel_res=cg["true_residual"] / np.sqrt(cg["u0"]),
                                trace5=cg["trace"][:5].tolist(),
                                seconds=time.time() - t0))
        print(res["runs"][-1], flush=True)
        if b == 128:
            dense_variants(a, rhs, n, b, res, xs)
            o = Oracle()
            o.set_symv_order(1)
            t0 = time.time()
            cgt = o.solve_cg(n, b, a, rhs, eps=1e-6, max_iters=500, recompute_interval=50)
            o.set_symv_order(0)
            xs["oracle_tile_partials_b128"] = unpad(cgt["x"], n)
            res["runs"].append(dict(variant="C restatement, tile partials, b=128",
                                    iterations=cgt["iterations"], u0=cgt["u0"],
                                    true_residual=cgt["true_residual"],
                                    rel_res=cgt["true_residual"] / np.sqrt(cgt["u0"]),
                                    trace5=cgt["trace"][:5].tolist(),
                                    seconds=time.time() - t0))
            print(res["runs"][-1], flush=True)
            o = fma_oracle()
            t0 = time.time()
            cgf = o.solve_cg(n, b, a, rhs, eps=1e-6, max_iters=500, recompute_interval=50)
            xs["oracle_fma_b128"] = unpad(cgf["x"], n)
            res["runs"].append(dict(variant="C restatement, FMA-contracted, b=128",
                                    iterations=cgf["iterations"], u0=cgf["u0"],
                                    true_residual=cgf["true_residual"],
                                    rel_res=cgf["true_residual"] / np.sqrt(cgf["u0"]),
                                    trace5=cgf["trace"][:5].tolist(),
                                    seconds=time.time() - t0))
            print(res["runs"][-1], flush=True)
        del a
    ref = xs.get("ref_b128")
    if ref is not None:
        res["x_rel_vs_ref_b128"] = {k: float(np.linalg.norm(v - ref) / np.linalg.norm(ref))
                                    for k, v in xs.items()}
    print(json.dumps(res))
    if args.out:
        with open(args.out, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
