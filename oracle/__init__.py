"""TEST INFRASTRUCTURE ONLY — the parity checker, never the product.

ctypes wrappers for
  * ``oracle/liboracle.so``  — the plain-C restatement of the reference
    (``hs_oracle.c``; every function cites reference file:line), and
  * ``oracle/_ref/libhsolve_ref.so`` — the UNMODIFIED reference sources from
    /root/reference/proj/src compiled by ``oracle/Makefile`` (present only
    where it was built; it travels to the GPU box as a prebuilt .so).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this package. The product
(``paper_2605_13209_b200``) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libhsolve_ref.so")
REF_ROOT = "/root/reference/proj"

_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_sz = C.c_size_t
_i64p = C.POINTER(C.c_int64)


def build(ref: bool | None = None) -> None:
    """Compile the oracle (always) and the reference (when its sources exist)."""
    subprocess.run(["make", "-s", "-C", HERE, "liboracle.so"], check=True)
    if ref is None:
        ref = os.path.isdir(os.path.join(REF_ROOT, "src"))
    if ref:
        subprocess.run(["make", "-s", "-j8", "-C", HERE, "ref"], check=True)


def nrows(n: int, b: int) -> int:
    return (n + b - 1) // b


def packed_len(n: int, b: int) -> int:
    N = nrows(n, b)
    return N * (N + 1) // 2 * b * b


class Oracle:
    """The C restatement (hs_oracle.h)."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build(ref=False)
        L = self.lib = C.CDLL(path)
        L.hso_rng_at.restype = C.c_uint64
        L.hso_rng_at.argtypes = [C.c_uint64, C.c_uint64]
        L.hso_uniform_pm1.restype = C.c_double
        L.hso_uniform_pm1.argtypes = [C.c_uint64, C.c_uint64]
        L.hso_generate_inputs.argtypes = [_sz, _sz, C.c_uint64, _dp]
        L.hso_median_pairwise_distance.restype = C.c_double
        L.hso_median_pairwise_distance.argtypes = [_dp, _sz, _sz]
        L.hso_generate_spd.argtypes = [_sz, _sz, C.c_double, C.c_double, C.c_double,
                                       _sz, C.c_uint64, C.c_int, _dp]
        L.hso_generate_rhs.argtypes = [_sz, _sz, C.c_uint64, _dp]
        L.hso_symv.argtypes = [_sz, _sz, _dp, _dp, _dp, C.c_int]
        L.hso_set_symv_order.argtypes = [C.c_int]
        L.hso_dot.restype = C.c_double
        L.hso_dot.argtypes = [_sz, _sz, _dp, _dp]
        L.hso_solve_cg.argtypes = [_sz, _sz, _dp, _dp, C.c_double, _sz, _sz, C.c_int,
                                   _dp, _dp, C.c_void_p, _sz, _i64p]
        L.hso_potf_block.argtypes = [_dp, _sz, _i64p]
        L.hso_trsm_block.argtypes = [_dp, _dp, _sz, _i64p]
        L.hso_gemm_update.argtypes = [_dp, _dp, _dp, _sz]
        L.hso_syrk_update.argtypes = [_dp, _dp, _sz]
        L.hso_factorize.argtypes = [_sz, _sz, _dp, C.c_int, _i64p, _i64p]
        L.hso_forward_substitute.argtypes = [_sz, _sz, _dp, _dp, _dp]
        L.hso_back_substitute.argtypes = [_sz, _sz, _dp, _dp, _dp]
        L.hso_solve_spd.argtypes = [_sz, _sz, _dp, _dp, C.c_int, _dp, _dp, _i64p, _i64p]
        L.hso_partition_for_fraction.restype = _sz
        L.hso_partition_for_fraction.argtypes = [C.c_double, _sz]
        L.hso_cholesky_border.restype = _sz
        L.hso_cholesky_border.argtypes = [C.c_double, _sz, _sz]

    # -- assembly ---------------------------------------------------------
    def generate_inputs(self, n, dim=2, seed=42):
        out = np.empty(n * dim)
        assert self.lib.hso_generate_inputs(n, dim, seed, out) == 0
        return out

    def median_pairwise_distance(self, pts, n, dim=2):
        return self.lib.hso_median_pairwise_distance(np.ascontiguousarray(pts), n, dim)

    def generate_spd(self, n, b, seed=42, sigma_f2=1.0, length_scale=0.0,
                     sigma_n2=1e-2, dim=2, threads=None):
        out = np.zeros(packed_len(n, b))
        st = self.lib.hso_generate_spd(n, b, sigma_f2, length_scale, sigma_n2, dim,
                                       seed, threads or os.cpu_count(), out)
        if st:
            raise ValueError(f"generate_spd status {st}")
        return out

    def generate_rhs(self, n, b, seed=42):
        out = np.zeros(nrows(n, b) * b)
        self.lib.hso_generate_rhs(n, b, seed, out)
        return out

    # -- CG -----------------------------------------------------------------
    def symv(self, n, b, a, x, threads=None):
        y = np.zeros(nrows(n, b) * b)
        self.lib.hso_symv(n, b, a, np.ascontiguousarray(x), y, threads or os.cpu_count())
        return y

    def set_symv_order(self, order: int) -> None:
        """0 = the reference's accumulation order; 1 = per-tile partials
        (the GPU SYMV's class) — for the iteration-envelope tests only."""
        self.lib.hso_set_symv_order(int(order))

    def dot(self, n, b, u, v):
        return self.lib.hso_dot(n, b, u, v)

    def solve_cg(self, n, b, a, rhs, eps=1e-6, max_iters=500, recompute_interval=50,
                 threads=None, trace=True):
        x = np.zeros(nrows(n, b) * b)
        stats = np.zeros(5)
        tr = np.zeros(3 * max(max_iters, 1)) if trace else None
        err = C.c_int64(-1)
        st = self.lib.hso_solve_cg(n, b, a, rhs, eps, max_iters, recompute_interval,
                                   threads or os.cpu_count(), x, stats,
                                   tr.ctypes.data if tr is not None else None,
                                   max_iters if trace else 0, C.byref(err))
        it = int(stats[0])
        return dict(status=st, x=x, iterations=it, recomputations=int(stats[1]),
                    converged=bool(stats[2]), u0=stats[3], true_residual=stats[4],
                    trace=(tr[: 3 * it].reshape(-1, 3) if tr is not None else None),
                    err_iter=err.value)

    # -- Cholesky -------------------------------------------------------------
    def factorize(self, n, b, a, threads=None):
        """In place on a copy; returns (status, L, block_row, pivot)."""
        L = np.array(a, dtype=np.float64, copy=True)
        r, p = C.c_int64(-1), C.c_int64(-1)
        st = self.lib.hso_factorize(n, b, L, threads or os.cpu_count(), C.byref(r), C.byref(p))
        return st, L, r.value, p.value

    def forward_substitute(self, n, b, l, rhs):
        y = np.zeros(nrows(n, b) * b)
        st = self.lib.hso_forward_substitute(n, b, l, rhs, y)
        return st, y

    def back_substitute(self, n, b, l, y):
        x = np.zeros(nrows(n, b) * b)
        st = self.lib.hso_back_substitute(n, b, l, y, x)
        return st, x

    def solve_spd(self, n, b, a, rhs, threads=None):
        L = np.array(a, copy=True)
        x = np.zeros(nrows(n, b) * b)
        stats = np.zeros(1)
        r, p = C.c_int64(-1), C.c_int64(-1)
        st = self.lib.hso_solve_spd(n, b, L, rhs, threads or os.cpu_count(), x, stats,
                                    C.byref(r), C.byref(p))
        return dict(status=st, x=x, L=L, true_residual=stats[0], block_row=r.value,
                    pivot=p.value)

    def partition_for_fraction(self, f, rows):
        return self.lib.hso_partition_for_fraction(f, rows)

    def cholesky_border(self, f, col, rows):
        return self.lib.hso_cholesky_border(f, col, rows)


class Reference:
    """The real reference (oracle/_ref/libhsolve_ref.so via oracle/ref_capi.cpp)."""

    @staticmethod
    def available() -> bool:
        return os.path.exists(REF_SO)

    def __init__(self, path: str = REF_SO):
        L = self.lib = C.CDLL(path)
        L.ref_generate_spd.argtypes = [_sz, _sz, C.c_double, C.c_double, C.c_double, _sz,
                                       C.c_uint64, _dp]
        L.ref_generate_inputs.argtypes = [_sz, _sz, C.c_uint64, _dp]
        L.ref_median_pairwise_distance.restype = C.c_double
        L.ref_median_pairwise_distance.argtypes = [_dp, _sz, _sz]
        L.ref_generate_rhs.argtypes = [_sz, _sz, C.c_uint64, _dp]
        L.ref_symv.argtypes = [_sz, _sz, _dp, _dp, _dp]
        L.ref_solve_cg.argtypes = [_sz, _sz, _dp, _dp, C.c_double, _sz, _sz, C.c_double, _sz,
                                   _dp, _dp, C.c_void_p, _sz, C.c_void_p]
        L.ref_factorize.argtypes = [_sz, _sz, _dp, C.c_double, _sz, C.c_void_p,
                                    C.POINTER(C.c_longlong), C.POINTER(C.c_longlong)]
        L.ref_solve_spd.argtypes = [_sz, _sz, _dp, _dp, C.c_double, _sz, _dp, _dp]
        L.ref_forward_substitute.argtypes = [_sz, _sz, _dp, _dp, _dp]
        L.ref_back_substitute.argtypes = [_sz, _sz, _dp, _dp, _dp]
        L.ref_potf_block.argtypes = [_dp, _sz, C.POINTER(C.c_longlong)]
        L.ref_trsm_block.argtypes = [_dp, _dp, _sz]
        L.ref_gemm_update.argtypes = [_dp, _dp, _dp, _sz]
        L.ref_syrk_update.argtypes = [_dp, _dp, _sz]
        L.ref_partition_for_fraction.restype = _sz
        L.ref_partition_for_fraction.argtypes = [C.c_double, _sz]
        L.ref_cholesky_border.restype = _sz
        L.ref_cholesky_border.argtypes = [C.c_double, _sz, _sz]
        L.ref_save_matrix.argtypes = [_sz, _sz, _dp, C.c_char_p]
        L.ref_load_matrix.argtypes = [C.c_char_p, C.POINTER(_sz), C.POINTER(_sz), C.c_void_p,
                                      _sz, _i64p, _i64p]
        L.ref_save_vector.argtypes = [_sz, _sz, _dp, C.c_char_p]

    # matrix_io.hpp:16-19
    def save_matrix(self, n, b, a, path):
        st = self.lib.ref_save_matrix(n, b, np.ascontiguousarray(a), os.fsencode(path))
        assert st == 0, st

    def load_matrix(self, path):
        """(status, n, b, values | None, expected, actual)."""
        n, b = _sz(), _sz()
        ea, eb = C.c_int64(-1), C.c_int64(-1)
        st = self.lib.ref_load_matrix(os.fsencode(path), C.byref(n), C.byref(b), None, 0,
                                      C.byref(ea), C.byref(eb))
        if st != 0:
            return st, 0, 0, None, ea.value, eb.value
        out = np.empty(packed_len(n.value, b.value))
        st = self.lib.ref_load_matrix(os.fsencode(path), C.byref(n), C.byref(b),
                                      out.ctypes.data, out.size, C.byref(ea), C.byref(eb))
        return st, n.value, b.value, out, -1, -1

    def save_vector(self, n, b, v, path):
        st = self.lib.ref_save_vector(n, b, np.ascontiguousarray(v), os.fsencode(path))
        assert st == 0, st

    def generate_spd(self, n, b, seed=42, sigma_f2=1.0, length_scale=0.0, sigma_n2=1e-2, dim=2):
        out = np.zeros(packed_len(n, b))
        st = self.lib.ref_generate_spd(n, b, sigma_f2, length_scale, sigma_n2, dim, seed, out)
        if st:
            raise ValueError(f"ref generate_spd status {st}")
        return out

    def generate_inputs(self, n, dim=2, seed=42):
        out = np.empty(n * dim)
        self.lib.ref_generate_inputs(n, dim, seed, out)
        return out

    def generate_rhs(self, n, b, seed=42):
        out = np.zeros(nrows(n, b) * b)
        self.lib.ref_generate_rhs(n, b, seed, out)
        return out

    def symv(self, n, b, a, x):
        y = np.zeros(nrows(n, b) * b)
        self.lib.ref_symv(n, b, a, np.ascontiguousarray(x), y)
        return y

    def solve_cg(self, n, b, a, rhs, eps=1e-6, max_iters=500, recompute_interval=50,
                 fraction=0.0, workers=None, trace=True):
        x = np.zeros(nrows(n, b) * b)
        stats = np.zeros(8)
        tr = np.zeros(3 * max(max_iters, 1)) if trace else None
        led = np.zeros(4, dtype=np.uint64)
        st = self.lib.ref_solve_cg(n, b, a, rhs, eps, max_iters, recompute_interval, fraction,
                                   workers or os.cpu_count(), x, stats,
                                   tr.ctypes.data if tr is not None else None,
                                   max_iters if trace else 0, led.ctypes.data)
        it = int(stats[0])
        return dict(status=st, x=x, iterations=it, recomputations=int(stats[1]),
                    converged=bool(stats[2]), u0=stats[3], true_residual=stats[4],
                    wall_ms=stats[5], compute_ms=stats[6], split_row=int(stats[7]),
                    trace=(tr[: 3 * it].reshape(-1, 3) if tr is not None else None),
                    ledger=dict(scalar=int(led[0]), subvector=int(led[1]),
                                initial_matrix=int(led[2]), result=int(led[3])))

    def factorize(self, n, b, a, fraction=0.0, workers=None):
        L = np.array(a, copy=True)
        stats = np.zeros(2)
        r, p = C.c_longlong(-1), C.c_longlong(-1)
        st = self.lib.ref_factorize(n, b, L, fraction, workers or os.cpu_count(),
                                    stats.ctypes.data, C.byref(r), C.byref(p))
        return dict(status=st, L=L, factor_ms=stats[0], block_row=r.value, pivot=p.value)

    def solve_spd(self, n, b, a, rhs, fraction=0.0, workers=None):
        L = np.array(a, copy=True)
        x = np.zeros(nrows(n, b) * b)
        stats = np.zeros(5)
        st = self.lib.ref_solve_spd(n, b, L, rhs, fraction, workers or os.cpu_count(), x, stats)
        return dict(status=st, x=x, L=L, factor_ms=stats[0], solve_ms=stats[1],
                    wall_ms=stats[2], true_residual=stats[4])

    def forward_substitute(self, n, b, l, rhs):
        y = np.zeros(nrows(n, b) * b)
        return self.lib.ref_forward_substitute(n, b, l, rhs, y), y

    def back_substitute(self, n, b, l, y):
        x = np.zeros(nrows(n, b) * b)
        return self.lib.ref_back_substitute(n, b, l, y, x), x
