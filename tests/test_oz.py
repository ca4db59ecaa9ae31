"""Emulated-FP64 GEMM update on the INT8 tensor cores (Ozaki scheme I,
hs_oz_gemm_tiles): C -= P Q^T for b x b tiles, the Cholesky trailing-update
building block (gemm_update / syrk_update, block_kernels.cpp:39-57).

* exact mode: operands whose rows fit one 7-bit slice give a bit-exact
  result (integer arithmetic end to end);
* random and GP-like operands: error within the FP64 GEMM rounding bound
  2^-53 * K * |P||Q|^T (tolerance written below), slices = 8;
* lower_only (SYRK) leaves the strict upper triangle untouched.
"""
import numpy as np
import pytest
import torch

import paper_2605_13209_b200 as hs
from paper_2605_13209_b200 import hsolve as H

pytestmark = pytest.mark.gpu


def run_oz(rt, C, P, Q, slices=8, lower_only=False):
    b = C.shape[-1]
    dc, dp, dq = (torch.from_numpy(np.ascontiguousarray(x)).cuda() for x in (C, P, Q))
    H._check(rt._L.hs_oz_gemm_tiles(rt.ctx, dc.data_ptr(), dp.data_ptr(), dq.data_ptr(), b,
                                    C.shape[0], slices, int(lower_only)))
    return dc.cpu().numpy()


@pytest.mark.parametrize("b,count", [(128, 1), (256, 2), (512, 3)])
def test_exact_single_slice_operands(rt, b, count):
    rng = np.random.default_rng(b)
    # entries k * 2^-6 with |k| <= 63 and a 63 in every row: e = 0 after the
    # row max, so slice 1 holds k exactly and all other slices are zero
    P = rng.integers(-63, 64, size=(count, b, b)).astype(np.float64)
    Q = rng.integers(-63, 64, size=(count, b, b)).astype(np.float64)
    P[:, :, 0] = 63
    Q[:, :, 1] = -63
    P *= 2.0 ** -6
    Q *= 2.0 ** -6
    C = rng.integers(-1000, 1000, size=(count, b, b)).astype(np.float64)
    got = run_oz(rt, C, P, Q)
    want = C - np.einsum("tik,tjk->tij", P, Q)  # exact: integers / 2^12 < 2^53
    assert np.array_equal(got, want)


@pytest.mark.parametrize("b,count,slices", [(128, 2, 8), (512, 2, 8), (256, 1, 8)])
def test_random_operands_fp64_accuracy(rt, b, count, slices):
    rng = np.random.default_rng(7 + b)
    # rows with very different scales, signs, some zero rows
    P = rng.standard_normal((count, b, b)) * np.exp2(rng.integers(-30, 30, (count, b, 1)))
    Q = rng.standard_normal((count, b, b)) * np.exp2(rng.integers(-30, 30, (count, b, 1)))
    P[:, 3, :] = 0.0
    C = rng.standard_normal((count, b, b))
    got = run_oz(rt, C, P, Q, slices)
    ref = C - np.einsum("tik,tjk->tij", P.astype(np.longdouble), Q.astype(np.longdouble))
    bound = np.einsum("tik,tjk->tij", np.abs(P), np.abs(Q)) + np.abs(C)
    err = np.abs(got - ref.astype(np.float64))
    # FP64 GEMM worst-case rounding: K * 2^-53 * (|P||Q|^T + |C|)
    assert (err <= b * 2.0 ** -53 * bound + 1e-300).all(), (err / bound).max()
    # and far tighter on average
    assert np.median(err / np.maximum(bound, 1e-300)) < 2.0 ** -50


def test_gp_panel_update_matches_dmma(rt, oracle):
    # a real Cholesky panel: L_ij tiles of the factored GP matrix
    n, b = 2048, 512
    a = oracle.generate_spd(n, b, seed=42)
    st, L, _, _ = oracle.factorize(n, b, a)
    N = n // b
    tri = lambda i, j: (i * (i + 1) // 2 + j) * b * b
    P = np.stack([L[tri(2, 0):tri(2, 0) + b * b].reshape(b, b),
                  L[tri(3, 0):tri(3, 0) + b * b].reshape(b, b)])
    Q = np.stack([L[tri(3, 0):tri(3, 0) + b * b].reshape(b, b),
                  L[tri(3, 0):tri(3, 0) + b * b].reshape(b, b)])
    C = np.stack([a[tri(3, 2):tri(3, 2) + b * b].reshape(b, b),
                  a[tri(3, 3):tri(3, 3) + b * b].reshape(b, b)])
    got = run_oz(rt, C, P, Q)
    ref = C - np.einsum("tik,tjk->tij", P.astype(np.longdouble), Q.astype(np.longdouble))
    dm = C.copy()
    dc, dp, dq = (torch.from_numpy(np.ascontiguousarray(x)).cuda() for x in (dm, P, Q))
    H.gemm_update_tiles_device(rt, dc.data_ptr(), dp.data_ptr(), dq.data_ptr(), b, 2)
    dm = dc.cpu().numpy()
    e_oz = np.abs(got - ref.astype(np.float64)).max()
    e_dm = np.abs(dm - ref.astype(np.float64)).max()
    assert e_oz <= 4 * e_dm + 1e-15 * np.abs(C).max(), (e_oz, e_dm)


def test_lower_only_leaves_upper_triangle(rt):
    b = 256
    rng = np.random.default_rng(3)
    P = rng.standard_normal((1, b, b))
    C = rng.standard_normal((1, b, b))
    got = run_oz(rt, C, P, P, lower_only=True)
    full = C - np.einsum("tik,tjk->tij", P, P)
    il = np.tril_indices(b)
    iu = np.triu_indices(b, 1)
    assert np.array_equal(got[0][iu], C[0][iu])
    assert np.abs(got[0][il] - full[0][il]).max() <= 1e-12 * np.abs(full).max()


def test_nonfinite_rows_propagate_nan(rt):
    b = 128
    P = np.ones((1, b, b))
    Q = np.ones((1, b, b))
    P[0, 5, 7] = np.nan
    got = run_oz(rt, np.zeros((1, b, b)), P, Q)
    assert np.isnan(got[0, 5]).all() and np.isfinite(np.delete(got[0], 5, axis=0)).all()


# ---------------------------------------------------------------------------
# Cholesky with the trailing update on the INT8 tensor cores


def lower_mask(n, b):
    N = (n + b - 1) // b
    m = np.zeros(N * (N + 1) // 2 * b * b, dtype=bool)
    for i in range(N):
        for j in range(i + 1):
            t = np.ones((b, b), dtype=bool)
            if i == j:
                t = np.tril(t)
            m[(i * (i + 1) // 2 + j) * b * b:(i * (i + 1) // 2 + j + 1) * b * b] = t.ravel()
    return m


@pytest.mark.parametrize("n,b", [(1024, 128), (2048, 512), (1500, 256), (4096, 512)])
def test_cholesky_emulated_fp64_matches_oracle(oracle, n, b):
    rt = hs.Runtime()
    try:
        a = oracle.generate_spd(n, b, seed=42)
        st, L_ref, _, _ = oracle.factorize(n, b, a)
        mask = lower_mask(n, b)
        errs = {}
        for slices in (0, 8):
            rt.set_cholesky_gemm(slices)
            m = hs.DeviceMatrix(rt, n, b).upload(a)
            H.potrf_device(rt, m)
            got = m.download()
            errs[slices] = np.abs(got[mask] - L_ref[mask]).max()
            m.free()
        scale = np.abs(a[mask]).max()
        # the reference's cross-block-size bound (test_cholesky_solver.cpp:94-113)
        assert errs[8] <= 1e-10 * scale, errs
        # and no worse than the FP64 DMMA path's own distance to the oracle
        assert errs[8] <= 4 * errs[0] + 1e-14 * scale, errs
    finally:
        rt.close()


def test_cholesky_emulated_solve_and_not_spd(oracle):
    n, b = 2048, 256
    rt = hs.Runtime()
    try:
        rt.set_cholesky_gemm(8)
        a = hs.generate_spd(n, b, seed=7)
        rhs = hs.generate_rhs(n, b, 7)
        res = hs.solve_spd(a.copy(), rhs, hs.SolverConfig(block_size=b), rt)
        ref = oracle.solve_spd(n, b, a.values, rhs.values)
        assert np.linalg.norm(res.x.values - ref["x"]) <= 1e-10 * np.linalg.norm(ref["x"])
        assert res.stats.true_residual <= 1e-10 * np.linalg.norm(rhs.values)
        bad = a.copy()
        bad.set(2 * b + 8, 2 * b + 8, -5.0)  # block row 2, pivot 8
        with pytest.raises(hs.NotSpdError) as ei:
            hs.factorize(bad, hs.SolverConfig(block_size=b), rt)
        assert ei.value.block_row == 2 and ei.value.pivot_index == 8
        with pytest.raises(hs.ConfigError):
            rt.set_cholesky_gemm(9)
    finally:
        rt.close()


@pytest.mark.parametrize("n,b", [(2048, 512), (1536, 128)])
def test_distributed_cholesky_emulated_world1(oracle, n, b):
    """The 2D block-cyclic NCCL path with the INT8-emulated update (panel
    broadcast into the contiguous buffer, sliced there; owned-pair lists)."""
    rt = hs.Runtime.distributed(0, 0, 1, hs.Runtime.nccl_unique_id())
    try:
        rt.set_cholesky_gemm(8)
        a = oracle.generate_spd(n, b, seed=42)
        st, L_ref, _, _ = oracle.factorize(n, b, a)
        m = hs.DeviceMatrix(rt, n, b, cyclic=True).upload(a)
        H.potrf_device(rt, m)
        mask = lower_mask(n, b)
        err = np.abs(m.download()[mask] - L_ref[mask]).max()
        assert err <= 1e-10 * np.abs(a[mask]).max(), err
    finally:
        rt.close()
