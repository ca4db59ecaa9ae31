"""GPU parity: the B200 kernels (through the C ABI) against the CPU oracle.

The oracle (oracle/hs_oracle.c) is bitwise identical to the reference
(tests/test_oracle.py pins that); these tests compare the CUDA path with it on
the same seeded inputs. Tolerances (written next to each check):

* assembly: elementwise relative <= 4 ulp (only exp differs; d2 is computed
  with the reference's mul-then-add rounding); diagonal and padding exact.
* SYMV: |y - y_cpu| <= 1e-13 * (|A| |x|)_i  (summation order only).
* CG: |iters - iters_cpu| <= 2; ||x - x_cpu|| / ||x_cpu|| <= 1e-6;
  true residual <= 2 eps sqrt(u0) (test_cg_solver.cpp:88-89); trace
  iterations 1-5 within 1e-10 relative (the trace is chaotic after ~8).
* Cholesky: |L - L_cpu| <= 1e-10 max|A| (test_cholesky_solver.cpp:72-92);
  ||x - x_cpu|| / ||x_cpu|| <= 1e-10; ||b - Ax|| <= 1e-10 ||b||.
"""
import numpy as np
import pytest
import torch

import paper_2605_13209_b200 as hs
from paper_2605_13209_b200 import hsolve as H

pytestmark = pytest.mark.gpu

EPS = np.finfo(np.float64).eps


def dev(v: np.ndarray) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(v)).to("cuda")


def lower_mask(n, b):
    """Boolean mask over the packed array: True for canonical lower entries."""
    N = (n + b - 1) // b
    masks = []
    for i in range(N):
        for j in range(i + 1):
            m = np.ones((b, b), dtype=bool) if i != j else np.tril(np.ones((b, b), dtype=bool))
            masks.append(m.ravel())
    return np.concatenate(masks)


# ---------------------------------------------------------------------------
# (1) GP assembly


@pytest.mark.parametrize("n,b", [(45, 8), (1024, 128), (1000, 64), (300, 1), (2048, 512),
                                 (777, 256)])
def test_assembly_matches_oracle(rt, oracle, n, b):
    got = hs.generate_spd(n, b, seed=17, rt=rt).values
    ref = oracle.generate_spd(n, b, seed=17)
    exact = (ref == 1.0) | (ref == 0.0) | (ref == 1.01)  # padding / diagonal
    assert np.array_equal(got[exact], ref[exact])
    rel = np.abs(got - ref) / np.maximum(np.abs(ref), 1e-300)
    assert rel.max() <= 4 * EPS, rel.max()


def test_assembly_structure(rt):
    # test_genmat.cpp:51-66
    p = hs.KernelParams()
    m = hs.generate_spd(50, 8, p, 11, rt=rt)
    for q in range(0, 50, 7):
        assert m.element(q, q) == p.sigma_f2 + p.sigma_n2
    for r in range(0, 50, 5):
        for c in range(0, 50, 3):
            assert m.element(r, c) == m.element(c, r)
            if r != c:
                assert 0.0 < m.element(r, c) <= p.sigma_f2


def test_assembly_rejects_bad_variance(rt):
    with pytest.raises(hs.ConfigError):
        hs.generate_spd(16, 4, hs.KernelParams(sigma_f2=0.0), 1, rt=rt)


# ---------------------------------------------------------------------------
# (2) SYMV


@pytest.mark.parametrize("n,b", [(45, 8), (1024, 128), (1000, 64), (4096, 256), (2048, 512),
                                 (333, 7), (96, 32), (8192, 128),
                                 # work-unit edge cases: one tile, fewer units
                                 # than SMs, ragged last block row, many units
                                 (128, 128), (64, 64), (200, 128), (1300, 128),
                                 (12345, 128), (700, 64), (20000, 64), (1500, 256),
                                 (5000, 512)])
def test_symv_matches_oracle(rt, oracle, n, b):
    a = oracle.generate_spd(n, b, seed=5)
    x = oracle.generate_rhs(n, b, seed=9)
    y_ref = oracle.symv(n, b, a, x)
    m = hs.DeviceMatrix(rt, n, b).upload(a)
    dx, dy = dev(x), torch.zeros_like(dev(x))
    H.symv_device(rt, m, dx.data_ptr(), dy.data_ptr())
    y = dy.cpu().numpy()
    dense = hs.BlockedSPDMatrix(n, b, a).to_dense()
    scale = np.abs(dense) @ np.abs(x[:n]) + 1e-300
    err = np.abs(y[:n] - y_ref[:n]) / scale
    assert err.max() <= 1e-13, err.max()
    assert np.all(y[n:] == x[n:])  # identity padding: padded rows copy x (zeros)


@pytest.mark.parametrize("n,b", [(32768, 128), (8192, 512), (3000, 64)])
def test_symv_bitwise_deterministic_under_dynamic_units(rt, n, b):
    # the SYMV's work units are claimed dynamically (the CTA that processes
    # a unit varies run to run), but every partial slot belongs to a unit and
    # the finalize adds them in a fixed order: repeated products, and whole
    # CG solves, must be bitwise identical
    m = hs.generate_spd_device(rt, n, b, seed=7)
    g = torch.Generator(device="cuda").manual_seed(1)
    N = (n + b - 1) // b
    x = torch.randn(N * b, dtype=torch.float64, device="cuda", generator=g)
    x[n:] = 0
    ys = []
    for _ in range(4):
        y = torch.empty_like(x)
        H.symv_device(rt, m, x.data_ptr(), y.data_ptr())
        ys.append(y)
    for y in ys[1:]:
        assert torch.equal(y, ys[0])
    rhs = x.clone()
    sols = []
    for _ in range(2):
        out = torch.zeros_like(rhs)
        st = hs.solve_cg_device(rt, m, rhs.data_ptr(), out.data_ptr(),
                                hs.SolverConfig(block_size=b, eps=1e-300, max_iters=60))
        sols.append((out, st.true_residual))
    assert torch.equal(sols[0][0], sols[1][0]) and sols[0][1] == sols[1][1]
    m.free()


def test_symv_identity_and_worked_example(rt):
    # test_block_kernels.cpp:197-220
    ident = hs.BlockedSPDMatrix.identity(13, 4)
    x = np.zeros(16)
    x[:13] = np.arange(1, 14) * 0.5
    m = hs.DeviceMatrix(rt, 13, 4).upload(ident)
    dx = dev(x)
    dy = torch.zeros_like(dx)
    H.symv_device(rt, m, dx.data_ptr(), dy.data_ptr())
    assert np.array_equal(dy.cpu().numpy(), x)
    w = hs.BlockedSPDMatrix(2, 1)
    w.set(0, 0, 2.0)
    w.set(1, 0, 1.0)
    w.set(1, 1, 3.0)
    m2 = hs.DeviceMatrix(rt, 2, 1).upload(w)
    dx = dev(np.array([1.0, 1.0]))
    dy = torch.zeros_like(dx)
    H.symv_device(rt, m2, dx.data_ptr(), dy.data_ptr())
    assert dy.cpu().tolist() == [3.0, 4.0]


def test_symv_ignores_stale_upper_halves(rt, oracle):
    n, b = 512, 128
    a = oracle.generate_spd(n, b, seed=3)
    x = oracle.generate_rhs(n, b, seed=4)
    y_ref = oracle.symv(n, b, a, x)
    poisoned = a.copy()
    mask = lower_mask(n, b)
    poisoned[~mask] = np.nan  # strict upper halves of diagonal tiles
    m = hs.DeviceMatrix(rt, n, b).upload(poisoned)
    dx = dev(x)
    dy = torch.zeros_like(dx)
    H.symv_device(rt, m, dx.data_ptr(), dy.data_ptr())
    y = dy.cpu().numpy()
    assert np.all(np.isfinite(y))
    assert np.abs(y - y_ref).max() <= 1e-12 * np.abs(y_ref).max()


# ---------------------------------------------------------------------------
# (3) CG


@pytest.mark.parametrize("n,b", [(1024, 128), (1000, 64), (2048, 512), (1024, 32), (257, 16)])
def test_cg_matches_oracle(rt, oracle, n, b):
    a = oracle.generate_spd(n, b, seed=42)
    rhs = oracle.generate_rhs(n, b, seed=42)
    ref = oracle.solve_cg(n, b, a, rhs, eps=1e-6, max_iters=500)
    cfg = hs.SolverConfig(block_size=b, record_trace=True)
    res = hs.solve_cg(hs.BlockedSPDMatrix(n, b, a), hs.BlockVector(n, b, rhs), cfg, rt)
    st = res.stats
    assert st.converged and ref["converged"]
    assert abs(st.iterations - ref["iterations"]) <= 2
    x, xr = res.x.values[:n], ref["x"][:n]
    assert np.linalg.norm(x - xr) <= 1e-6 * np.linalg.norm(xr)
    assert st.true_residual <= 2 * cfg.eps * np.sqrt(st.u0)
    assert abs(st.u0 - ref["u0"]) <= 1e-14 * ref["u0"]
    tr = np.array([[t.u, t.alpha, t.beta] for t in st.trace[:5]])
    assert np.allclose(tr, ref["trace"][:5], rtol=1e-10, atol=0)
    assert np.all(res.x.values[n:] == 0.0)


def test_cg_identity_one_iteration(rt):
    # test_cg_solver.cpp:28-39
    ident = hs.BlockedSPDMatrix.identity(64, 16)
    rhs = hs.generate_rhs(64, 16, 1)
    res = hs.solve_cg(ident, rhs, hs.SolverConfig(block_size=16), rt)
    assert res.stats.iterations == 1 and res.stats.converged
    assert np.array_equal(res.x.values, rhs.values)


def test_cg_zero_rhs(rt):
    # test_cg_solver.cpp:41-51
    ident = hs.BlockedSPDMatrix.identity(16, 4)
    res = hs.solve_cg(ident, hs.BlockVector(16, 4), hs.SolverConfig(block_size=4), rt)
    assert res.stats.iterations == 0 and res.stats.converged and res.stats.u0 == 0.0
    assert np.all(res.x.values == 0.0)


def test_cg_small_system_vs_dense_solve(rt, oracle):
    # test_cg_solver.cpp:53-74
    n, b = 8, 2
    a = hs.BlockedSPDMatrix(n, b, oracle.generate_spd(n, b, seed=77))
    rhs = hs.BlockVector(n, b, oracle.generate_rhs(n, b, seed=77))
    x_direct = np.linalg.solve(a.to_dense(), rhs.logical())
    res = hs.solve_cg(a, rhs, hs.SolverConfig(block_size=b, eps=1e-10, max_iters=100), rt)
    assert res.stats.converged
    assert np.linalg.norm(res.x.logical() - x_direct) <= 1e-5 * np.linalg.norm(x_direct)


@pytest.mark.parametrize("n", [96, 256])
def test_cg_true_residual_bound(rt, oracle, n):
    # test_cg_solver.cpp:76-91
    b = 16
    a = hs.BlockedSPDMatrix(n, b, oracle.generate_spd(n, b, seed=13))
    rhs = hs.BlockVector(n, b, oracle.generate_rhs(n, b, seed=13))
    cfg = hs.SolverConfig(block_size=b, eps=1e-6, max_iters=2000)
    st = hs.solve_cg(a, rhs, cfg, rt).stats
    assert st.converged and st.u0 > 0
    assert st.true_residual <= 2 * cfg.eps * np.sqrt(st.u0)


def test_cg_recompute_cadence(rt, oracle):
    # test_cg_solver.cpp:150-161, 219-234
    n, b = 128, 16
    a = hs.BlockedSPDMatrix(n, b, oracle.generate_spd(n, b, seed=21))
    rhs = hs.BlockVector(n, b, oracle.generate_rhs(n, b, seed=21))
    cfg = hs.SolverConfig(block_size=b, recompute_interval=5, eps=1e-300, max_iters=12)
    st = hs.solve_cg(a, rhs, cfg, rt).stats
    assert st.iterations == 12 and st.recomputations == 2
    cfg = hs.SolverConfig(block_size=b, recompute_interval=3, eps=1e-8, max_iters=500)
    a6 = hs.BlockedSPDMatrix(96, b, oracle.generate_spd(96, b, seed=6))
    r6 = hs.BlockVector(96, b, oracle.generate_rhs(96, b, seed=6))
    st = hs.solve_cg(a6, r6, cfg, rt).stats
    assert st.converged and st.recomputations == st.iterations // 3
    assert st.true_residual <= 2 * cfg.eps * np.sqrt(st.u0)


def test_cg_iteration_cap_is_a_status(rt, oracle):
    # test_cg_solver.cpp:236-248
    n, b = 64, 16
    a = hs.BlockedSPDMatrix(n, b, oracle.generate_spd(n, b, seed=14))
    rhs = hs.BlockVector(n, b, oracle.generate_rhs(n, b, seed=14))
    st = hs.solve_cg(a, rhs, hs.SolverConfig(block_size=b, eps=1e-14, max_iters=2), rt).stats
    assert not st.converged and st.iterations == 2


def test_cg_single_block_row(rt, oracle):
    # test_cg_solver.cpp:204-217
    a = hs.BlockedSPDMatrix(8, 8, oracle.generate_spd(8, 8, seed=2))
    rhs = hs.BlockVector(8, 8, oracle.generate_rhs(8, 8, seed=2))
    st = hs.solve_cg(a, rhs, hs.SolverConfig(block_size=8, eps=1e-10, max_iters=100), rt).stats
    assert st.converged and st.true_residual <= 1e-8


def test_cg_nonfinite_and_shape_errors(rt):
    # test_cg_solver.cpp:250-264
    ident = hs.BlockedSPDMatrix.identity(8, 4)
    rhs = hs.BlockVector(8, 4)
    rhs[3] = np.inf
    with pytest.raises(hs.NumericalError):
        hs.solve_cg(ident, rhs, hs.SolverConfig(block_size=4), rt)
    with pytest.raises(hs.ConfigError):
        hs.solve_cg(ident, hs.BlockVector(8, 2), hs.SolverConfig(block_size=4), rt)


def test_cg_device_resident_matches_host_entry(rt, oracle):
    n, b = 2048, 128
    m = hs.generate_spd_device(rt, n, b, seed=42)
    rhs = oracle.generate_rhs(n, b, seed=42)
    d_rhs = dev(rhs)
    d_x = torch.zeros_like(d_rhs)
    cfg = hs.SolverConfig(block_size=b, eps=1e-6)
    st = hs.solve_cg_device(rt, m, d_rhs.data_ptr(), d_x.data_ptr(), cfg)
    host = hs.solve_cg(m.to_host(), hs.BlockVector(n, b, rhs), cfg, rt)
    assert st.iterations == host.stats.iterations
    assert np.array_equal(d_x.cpu().numpy(), host.x.values)  # deterministic


# ---------------------------------------------------------------------------
# (4) Cholesky


@pytest.mark.parametrize("n,b", [(1024, 128), (2048, 512), (1000, 256), (1200, 384), (256, 32),
                                 (100, 16), (45, 8), (2, 1), (700, 96)])
def test_factor_and_solve_match_oracle(rt, oracle, n, b):
    a = oracle.generate_spd(n, b, seed=42)
    rhs = oracle.generate_rhs(n, b, seed=42)
    st, L_ref, _, _ = oracle.factorize(n, b, a)
    assert st == 0
    mask = lower_mask(n, b)
    work = hs.BlockedSPDMatrix(n, b, a.copy())
    hs.factorize(work, hs.SolverConfig(block_size=b), rt)
    maxa = np.abs(a[mask]).max()
    assert np.abs(work.values[mask] - L_ref[mask]).max() <= 1e-10 * maxa
    res = hs.solve_spd(hs.BlockedSPDMatrix(n, b, a.copy()), hs.BlockVector(n, b, rhs),
                       hs.SolverConfig(block_size=b), rt)
    ref = oracle.solve_spd(n, b, a, rhs)
    x, xr = res.x.values[:n], ref["x"][:n]
    assert np.linalg.norm(x - xr) <= 1e-10 * np.linalg.norm(xr)
    assert res.stats.true_residual <= 1e-10 * np.linalg.norm(rhs[:n])


@pytest.mark.parametrize("n", [256, 512, 1024, 2048])
def test_factor_reconstruction_acceptance_grid(rt, oracle, n):
    # acceptance.cpp:84-110: ||A - L L^T||_F / ||A||_F <= 1e-12 over
    # n x b in {256..2048} x {16, 32, 64, 128}; and the factors of the same
    # matrix at different block sizes agree (test_cholesky_solver.cpp:94-113)
    dense = {}
    for b in (16, 32, 64, 128):
        a = hs.BlockedSPDMatrix(n, b, oracle.generate_spd(n, b, seed=42))
        A = a.to_dense()
        hs.factorize(a, hs.SolverConfig(block_size=b), rt)
        L = np.tril(a.to_dense())
        assert np.linalg.norm(A - L @ L.T) <= 1e-12 * np.linalg.norm(A), (n, b)
        dense[b] = (L, np.abs(A).max())
    L16, maxa = dense[16]
    for b in (32, 64, 128):
        assert np.abs(dense[b][0] - L16).max() <= 1e-10 * maxa, (n, b)


def test_factor_closed_form_and_identity(rt):
    # test_cholesky_solver.cpp:35-70
    m = hs.BlockedSPDMatrix(2, 1)
    m.set(0, 0, 4.0)
    m.set(1, 0, 2.0)
    m.set(1, 1, 3.0)
    hs.factorize(m, hs.SolverConfig(block_size=1), rt)
    assert m.block(0, 0)[0, 0] == 2.0 and m.block(1, 0)[0, 0] == 1.0
    assert abs(m.block(1, 1)[0, 0] - np.sqrt(2.0)) <= 1e-15
    ident = hs.BlockedSPDMatrix.identity(12, 4)
    hs.factorize(ident, hs.SolverConfig(block_size=4), rt)
    for p in range(12):
        for q in range(p + 1):
            assert ident.element(p, q) == (1.0 if p == q else 0.0)


def test_not_spd_reports_column_and_pivot(rt, oracle):
    # test_cholesky_solver.cpp:208-224
    a = hs.BlockedSPDMatrix(64, 16, oracle.generate_spd(64, 16, seed=2))
    a.set(40, 40, -5.0)
    with pytest.raises(hs.NotSpdError) as ei:
        hs.factorize(a, hs.SolverConfig(block_size=16), rt)
    assert ei.value.block_row == 2 and ei.value.pivot_index == 40 % 16


def test_not_spd_dmma_path(rt, oracle):
    n, b = 1024, 128
    a = hs.BlockedSPDMatrix(n, b, oracle.generate_spd(n, b, seed=2))
    a.set(700, 700, -5.0)
    with pytest.raises(hs.NotSpdError) as ei:
        hs.factorize(a, hs.SolverConfig(block_size=b), rt)
    assert ei.value.block_row == 700 // b and ei.value.pivot_index == 700 % b


def test_substitutions(rt, oracle):
    # test_cholesky_solver.cpp:226-282
    ident = hs.BlockedSPDMatrix.identity(10, 4)
    rhs = hs.BlockVector(10, 4, np.arange(1, 11) * 0.5)
    y = hs.forward_substitute(ident, rhs, rt)
    x = hs.back_substitute(ident, y, rt)
    assert np.array_equal(y.logical(), rhs.logical()) and np.array_equal(x.logical(), rhs.logical())
    l2 = hs.BlockedSPDMatrix(2, 1)
    l2.set(0, 0, 2.0)
    l2.set(1, 0, 1.0)
    l2.set(1, 1, np.sqrt(2.0))
    r2 = hs.BlockVector(2, 1, np.array([2.0, 1.0 + np.sqrt(2.0)]))
    y = hs.forward_substitute(l2, r2, rt)
    assert np.allclose(y.logical(), [1.0, 1.0], rtol=1e-15)
    x = hs.back_substitute(l2, y, rt)
    a = np.array([[4.0, 2.0], [2.0, 3.0]])
    assert np.abs(a @ x.logical() - r2.logical()).max() <= 1e-12
    sing = hs.BlockedSPDMatrix.identity(4, 2)
    sing.set(2, 2, 0.0)
    r = hs.BlockVector(4, 2)
    r[0] = 1.0
    with pytest.raises(hs.SingularBlockError):
        hs.forward_substitute(sing, r, rt)
    with pytest.raises(hs.SingularBlockError):
        hs.back_substitute(sing, r, rt)


def test_singular_factor_dmma_path(rt):
    sing = hs.BlockedSPDMatrix.identity(300, 128)
    sing.set(130, 130, 0.0)
    r = hs.BlockVector(300, 128)
    r[0] = 1.0
    with pytest.raises(hs.SingularBlockError):
        hs.forward_substitute(sing, r, rt)


@pytest.mark.parametrize("n,b", [(1024, 128), (2048, 512), (200, 16), (1500, 256),
                                 (1152, 384), (700, 100), (999, 37), (2048, 1024)])
def test_substitutions_match_oracle(rt, oracle, n, b):
    # b = 128 f (f <= 4): staged cluster diagonal solve; 1024: unstaged (f = 8);
    # 100 / 16: cb = b; 37: odd b (scalar update path)
    a = oracle.generate_spd(n, b, seed=8)
    _, L, _, _ = oracle.factorize(n, b, a)
    rhs = oracle.generate_rhs(n, b, seed=8)
    _, y_ref = oracle.forward_substitute(n, b, L, rhs)
    _, x_ref = oracle.back_substitute(n, b, L, y_ref)
    lm = hs.BlockedSPDMatrix(n, b, L)
    y = hs.forward_substitute(lm, hs.BlockVector(n, b, rhs), rt)
    x = hs.back_substitute(lm, y, rt)
    assert np.linalg.norm(y.values - y_ref) <= 1e-11 * np.linalg.norm(y_ref)
    assert np.linalg.norm(x.values - x_ref) <= 1e-10 * np.linalg.norm(x_ref)


# ---------------------------------------------------------------------------
# single-tile kernels


@pytest.mark.parametrize("b", [1, 2, 5, 16, 32, 128, 512])
def test_potf_tiles_reconstruct(rt, oracle, b):
    # test_block_kernels.cpp:57-75
    rng = np.random.default_rng(11 + b)
    tiles = []
    for _ in range(3):
        mm = rng.uniform(-1, 1, (b, b))
        tiles.append(mm @ mm.T + b * np.eye(b))
    t = np.stack(tiles)
    d = dev(t)
    H.potf_tiles_device(rt, d.data_ptr(), b, 3)
    got = d.cpu().numpy()
    for k in range(3):
        ref = t[k].copy().ravel()
        assert oracle.lib.hso_potf_block(ref, b, None) == 0
        ref = ref.reshape(b, b)
        lo = np.tril(np.ones((b, b), dtype=bool))
        assert np.abs(got[k][lo] - ref[lo]).max() <= 1e-12 * np.abs(t[k]).max()
        assert np.array_equal(got[k][~lo], t[k][~lo])  # upper untouched


def test_potf_tile_not_spd(rt):
    d = dev(np.array([[1.0, 2.0], [2.0, 1.0]]))
    with pytest.raises(hs.NotSpdError) as ei:
        H.potf_tiles_device(rt, d.data_ptr(), 2, 1)
    assert ei.value.pivot_index == 1


@pytest.mark.parametrize("b,lower", [(128, False), (128, True), (256, False), (512, True),
                                     (16, False), (3, True)])
def test_gemm_update_tiles(rt, oracle, b, lower):
    rng = np.random.default_rng(b)
    cnt = 2
    c = rng.uniform(-1, 1, (cnt, b, b))
    p = rng.uniform(-1, 1, (cnt, b, b))
    q = p.copy() if lower else rng.uniform(-1, 1, (cnt, b, b))
    dc, dp, dq = dev(c), dev(p), dev(q)  # keep the operands alive
    H.gemm_update_tiles_device(rt, dc.data_ptr(), dp.data_ptr(), dq.data_ptr(), b, cnt, lower)
    got = dc.cpu().numpy()
    for k in range(cnt):
        ref = c[k].copy().ravel()
        if lower:
            oracle.lib.hso_syrk_update(ref, p[k].ravel().copy(), b)
        else:
            oracle.lib.hso_gemm_update(ref, p[k].ravel().copy(), q[k].ravel().copy(), b)
        ref = ref.reshape(b, b)
        assert np.abs(got[k] - ref).max() <= 1e-13 * b
        if lower:
            up = np.triu(np.ones((b, b), dtype=bool), 1)
            assert np.array_equal(got[k][up], c[k][up])


def test_gemm_worked_examples(rt):
    # test_block_kernels.cpp:150-183
    c = dev(np.array([[1.0, 0.0], [0.0, 1.0]]))
    p, q = dev(np.array([[1.0, 2.0], [3.0, 4.0]])), dev(np.eye(2))
    H.gemm_update_tiles_device(rt, c.data_ptr(), p.data_ptr(), q.data_ptr(), 2, 1)
    assert c.cpu().numpy().ravel().tolist() == [0.0, -2.0, -3.0, -3.0]
    c = dev(np.array([[5.0, 42.0], [2.0, 5.0]]))
    pp = dev(np.ones((2, 2)))
    H.gemm_update_tiles_device(rt, c.data_ptr(), pp.data_ptr(), pp.data_ptr(), 2, 1, True)
    assert c.cpu().numpy().ravel().tolist() == [3.0, 42.0, 0.0, 3.0]


def test_pageable_staged_upload_and_download(rt, oracle):
    # > 4 MB from pageable numpy memory takes the pinned staging threads
    # (hs_xfer.cu) both ways; the bytes must arrive unchanged
    n, b = 4096, 256
    a = oracle.generate_spd(n, b, seed=11)
    assert a.nbytes > (8 << 20)
    m = hs.DeviceMatrix(rt, n, b).upload(a)
    back = np.empty_like(a)
    m.download(back)
    assert back.tobytes() == a.tobytes()
    # odd sizes: a piece boundary inside a tile, a short tail
    n2, b2 = 3001, 200
    a2 = oracle.generate_spd(n2, b2, seed=12)
    m2 = hs.DeviceMatrix(rt, n2, b2).upload(a2)
    back2 = np.empty_like(a2)
    m2.download(back2)
    assert back2.tobytes() == a2.tobytes()
    m.free()
    m2.free()


def test_ctx_trim_releases_and_recovers(oracle):
    # hs_ctx_trim drops the cached upload, workspaces and staging buffers;
    # the next host-buffer call rebuilds them and gives the same answer
    rt = hs.Runtime()
    try:
        n, b = 1024, 128
        a = hs.BlockedSPDMatrix(n, b, oracle.generate_spd(n, b, seed=3))
        rhs = hs.BlockVector(n, b, oracle.generate_rhs(n, b, seed=3))
        cfg = hs.SolverConfig(block_size=b)
        first = hs.solve_cg(a, rhs, cfg, rt)
        free0 = torch.cuda.mem_get_info()[0]
        rt.trim()
        assert torch.cuda.mem_get_info()[0] > free0  # the cached upload is gone
        again = hs.solve_cg(a, rhs, cfg, rt)
        assert np.array_equal(first.x.values, again.x.values)
        rt.trim()
        rt.trim()  # idempotent
    finally:
        rt.close()


def test_kernel_launches_are_counted(rt):
    before = rt.kernel_launches()
    hs.generate_spd(256, 128, seed=1, rt=rt)
    assert rt.kernel_launches() > before


# ---------------------------------------------------------------------------
# distributed Cholesky path (2D block-cyclic + NCCL broadcasts), exercised on
# one GPU through a world-size-1 NCCL communicator


@pytest.mark.parametrize("n,b", [(1024, 128), (2048, 512), (1500, 256)])
def test_distributed_cholesky_world1_matches_oracle(oracle, n, b):
    rt = hs.Runtime.distributed(0, 0, 1, hs.Runtime.nccl_unique_id())
    try:
        a = oracle.generate_spd(n, b, seed=42)
        st, L_ref, _, _ = oracle.factorize(n, b, a)
        m = hs.DeviceMatrix(rt, n, b, cyclic=True).upload(a)
        H.potrf_device(rt, m)
        got = m.download()
        mask = lower_mask(n, b)
        assert np.abs(got[mask] - L_ref[mask]).max() <= 1e-10 * np.abs(a[mask]).max()
        # device-assembled cyclic matrix factors to the same L
        m2 = hs.generate_spd_device(rt, n, b, seed=42, cyclic=True)
        H.potrf_device(rt, m2)
        assert np.abs(m2.download()[mask] - L_ref[mask]).max() <= 1e-10 * np.abs(a[mask]).max()
        bad = a.copy()
        k = (0 * 1 // 2 + 0) * b * b + 5 * b + 5  # element (5, 5) of tile (0, 0)
        bad[k] = -1.0
        m3 = hs.DeviceMatrix(rt, n, b, cyclic=True).upload(bad)
        with pytest.raises(hs.NotSpdError) as ei:
            H.potrf_device(rt, m3)
        assert ei.value.block_row == 0 and ei.value.pivot_index == 5
    finally:
        rt.close()


@pytest.mark.parametrize("n,b", [(1024, 128), (2048, 512), (1500, 256)])
def test_distributed_solve_world1_matches_oracle(oracle, n, b):
    """Factor + substitutions + residual on a block-cyclic matrix through a
    world-1 communicator (the 1x1 grid takes the single-rank kernels)."""
    rt = hs.Runtime.distributed(0, 0, 1, hs.Runtime.nccl_unique_id())
    try:
        a = oracle.generate_spd(n, b, seed=42)
        rhs = oracle.generate_rhs(n, b, seed=42)
        ref = oracle.solve_spd(n, b, a, rhs)
        m = hs.DeviceMatrix(rt, n, b, cyclic=True).upload(a)
        orig = hs.DeviceMatrix(rt, n, b, cyclic=True).upload(a)
        d_rhs = dev(rhs)
        d_x = torch.zeros_like(d_rhs)
        sp = hs.solve_spd_device(rt, m, d_rhs.data_ptr(), d_x.data_ptr(), a_orig=orig)
        x = d_x.cpu().numpy()
        assert np.linalg.norm(x - ref["x"]) <= 1e-9 * np.linalg.norm(ref["x"])
        assert abs(sp.true_residual - ref["true_residual"]) <= 1e-10 * np.linalg.norm(rhs)
    finally:
        rt.close()


@pytest.mark.parametrize("n,b", [(2048, 128), (1000, 64)])
def test_distributed_cg_world1_matches_oracle(oracle, n, b):
    """The row-sharded NCCL protocol (reduce-scatter, all-gather of s,
    rank-ordered double-double dots) on one GPU via a world-1 communicator."""
    rt = hs.Runtime.distributed(0, 0, 1, hs.Runtime.nccl_unique_id())
    try:
        a = oracle.generate_spd(n, b, seed=42)
        rhs = oracle.generate_rhs(n, b, seed=42)
        ref = oracle.solve_cg(n, b, a, rhs, eps=1e-6, max_iters=500)
        m = hs.DeviceMatrix(rt, n, b).upload(a)
        d_rhs = dev(rhs)
        d_x = torch.zeros_like(d_rhs)
        st = hs.solve_cg_device(rt, m, d_rhs.data_ptr(), d_x.data_ptr(),
                                hs.SolverConfig(block_size=b, eps=1e-6))
        x = d_x.cpu().numpy()
        assert st.converged and abs(st.iterations - ref["iterations"]) <= 2
        assert np.linalg.norm(x[:n] - ref["x"][:n]) <= 1e-6 * np.linalg.norm(ref["x"][:n])
        assert st.true_residual <= 2e-6 * np.sqrt(st.u0)
    finally:
        rt.close()


@pytest.mark.parametrize("n,b", [(6144, 32), (4096, 128)])
def test_substitutions_wide_steps(rt, n, b):
    """Steps with many tiles (backward update without clusters, forward
    update grids of several waves) against a dense LAPACK-free reference:
    a diagonally dominant lower-triangular L solved by scipy."""
    from scipy.linalg import solve_triangular
    rng = np.random.default_rng(3)
    N = n // b
    dense = np.tril(rng.uniform(-1.0, 1.0, (n, n)) / np.sqrt(n))
    dense[np.diag_indices(n)] = rng.uniform(1.0, 2.0, n)
    ti, tj = np.tril_indices(N)
    packed = dense.reshape(N, b, N, b).transpose(0, 2, 1, 3)[ti, tj].ravel()
    rhs = rng.uniform(-1.0, 1.0, n)
    lm = hs.BlockedSPDMatrix(n, b, packed)
    y = hs.forward_substitute(lm, hs.BlockVector(n, b, rhs), rt)
    x = hs.back_substitute(lm, y, rt)
    y_ref = solve_triangular(dense, rhs, lower=True)
    x_ref = solve_triangular(dense.T, y_ref, lower=False)
    assert np.linalg.norm(y.logical() - y_ref) <= 1e-12 * np.linalg.norm(y_ref)
    assert np.linalg.norm(x.logical() - x_ref) <= 1e-12 * np.linalg.norm(x_ref)


@pytest.mark.parametrize("env", [{"HS_CG_PROG": "0"}, {"HS_CG_PROG": "0", "HS_CG_TAIL": "1"}],
                         ids=["memory_order_walk", "fused_tail"])
def test_cg_alternative_schedules_match_oracle(env):
    """The non-default CG schedules for b <= 128 -- the memory-order SYMV walk
    with a finalize kernel after it (HS_CG_PROG=0), and that walk with the
    fused single-launch tail (HS_CG_TAIL=1) -- meet the same oracle bounds as
    the default progressive path, in a subprocess (the switches are read
    once)."""
    import subprocess
    import sys
    code = r'''
import sys, numpy as np
sys.path.insert(0, ".")
import paper_2605_13209_b200 as hs
from oracle import Oracle
o = Oracle()
rt = hs.Runtime()
for n, b in [(1024, 128), (3000, 64), (2048, 512), (4096, 256)]:
    a = o.generate_spd(n, b, seed=11); rhs = o.generate_rhs(n, b, seed=11)
    ref = o.solve_cg(n, b, a, rhs, eps=1e-6)
    r = hs.solve_cg(hs.BlockedSPDMatrix(n, b, a), hs.BlockVector(n, b, rhs),
                    hs.SolverConfig(block_size=b, eps=1e-6, record_trace=True), rt)
    st = r.stats
    assert st.converged and abs(st.iterations - ref["iterations"]) <= max(2, 0.2 * ref["iterations"])
    assert st.true_residual <= 2e-6 * np.sqrt(st.u0)
    x = r.x.values[:n]
    assert np.linalg.norm(x - ref["x"][:n]) <= 1e-6 * np.linalg.norm(ref["x"][:n])
    tr = np.array([[t.u, t.alpha, t.beta] for t in st.trace[:5]])
    np.testing.assert_allclose(tr, ref["trace"][:5], rtol=1e-10)
print("TAIL OK")
'''
    import os
    env = dict(os.environ, **env)
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    p = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True,
                       text=True, timeout=600)
    assert p.returncode == 0 and "TAIL OK" in p.stdout, p.stdout + p.stderr


def test_split_tile_gemm_factor_bitwise_equals_128x128():
    """The default DMMA GEMM tiles (64x64 quadrants for C -= A B^T, 64x128 row
    halves for the in-place TRSM steps) give the same factor as 128x128 CTAs
    bit for bit -- every element sees the same K order and C - acc either way
    -- run after run (HS_GEMM64 is read once per process: subprocesses)."""
    import os
    import subprocess
    import sys
    code = r'''
import sys, os, numpy as np
sys.path.insert(0, ".")
import paper_2605_13209_b200 as hs
from paper_2605_13209_b200 import hsolve as H
rt = hs.Runtime()
out = []
for n, b in [(8192, 512), (4096, 256)]:
    m = hs.generate_spd_device(rt, n, b, seed=7)
    H.potrf_device(rt, m)
    L = m.download()
    N = n // b
    for i in range(N):
        t = i * (i + 1) // 2 + i
        T = L[t * b * b:(t + 1) * b * b].reshape(b, b)
        T[np.triu_indices(b, 1)] = 0.0  # the stale upper half is not part of L
    out.append(L)
np.save(sys.argv[1], np.concatenate(out))
'''
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = []
    for i, v in enumerate(["0", "1", "1"]):
        path = os.path.join("/tmp", f"hs_tiles_{os.getpid()}_{i}.npy")
        p = subprocess.run([sys.executable, "-c", code, path], cwd=root,
                           env=dict(os.environ, HS_GEMM64=v), capture_output=True,
                           text=True, timeout=600)
        assert p.returncode == 0, p.stdout + p.stderr
        res.append(np.load(path))
        os.remove(path)
    assert np.array_equal(res[0], res[1]) and np.array_equal(res[0], res[2])


def test_distributed_world1_factor_bitwise_equals_single_gpu():
    """At world 1 (1 x 1 grid) the block-cyclic factorization does the
    single-GPU path's work in the same order -- column pairs, K = 2b bulk
    updates over the broadcast panels, 64 x 64 CTA tiles beyond one wave --
    so the two factors agree bit for bit (n = 16384: the early bulk
    launches span many waves)."""
    import numpy as np
    n, b = 16384, 512
    rt1 = hs.Runtime()
    m = hs.generate_spd_device(rt1, n, b, seed=42)
    H.potrf_device(rt1, m)
    L1 = m.download()
    m.free()
    rtd = hs.Runtime.distributed(0, 0, 1, hs.Runtime.nccl_unique_id())
    md = hs.generate_spd_device(rtd, n, b, seed=42, cyclic=True)
    H.potrf_device(rtd, md)
    Ld = md.download()
    md.free()
    N = n // b
    for i in range(N):  # the diagonal tiles' upper halves are not part of L
        t = i * (i + 1) // 2 + i
        for L in (L1, Ld):
            T = L[t * b * b:(t + 1) * b * b].reshape(b, b)
            T[np.triu_indices(b, 1)] = 0.0
    assert np.array_equal(L1, Ld), float(np.abs(L1 - Ld).max())


@pytest.mark.parametrize("dist,slices", [(False, 0), (True, 0), (False, 8)])
def test_factor_bitwise_stable_under_outside_copy_traffic(dist, slices):
    """Unrelated copies on an independent stream beside the factorization
    (another library's work, an overlapped upload) leave the factor bitwise
    unchanged. Without the stage-release fence in the TMA-fed kernels
    (hs_chol.cu gemm_dmma_kernel) this reproduced wrong 64 x 64 tiles and
    NotSpd failures in most runs at this size, single-GPU and world-1
    distributed alike."""
    import numpy as np
    rt = (hs.Runtime.distributed(0, 0, 1, hs.Runtime.nccl_unique_id()) if dist
          else hs.Runtime())
    rt.set_cholesky_gemm(slices)  # 8: the INT8 tensor-core (Ozaki) trailing update
    n, b = 16384, 512

    def factor():
        m = hs.generate_spd_device(rt, n, b, seed=42, cyclic=dist)
        H.potrf_device(rt, m)
        L = m.download()
        m.free()
        return L

    ref = factor()
    a = torch.empty(32 << 20, dtype=torch.float64, device="cuda")  # 256 MB
    o = torch.empty_like(a)
    side = torch.cuda.Stream()
    for rep in range(3):
        with torch.cuda.stream(side):
            for _ in range(200):
                o.copy_(a)
        L = factor()
        torch.cuda.synchronize()
        assert np.array_equal(L, ref), f"rep {rep}: max diff {np.abs(L - ref).max()}"


@pytest.mark.parametrize("n,b", [(2048, 128), (1000, 64), (4096, 128)])
def test_cg_two_vector_recompute_matches_oracle(rt, oracle, n, b):
    """Recompute iterations on the progressive path (b <= 128) run A s and
    A x_old in one pass over A and form r = rhs - (A x_old + alpha A s)
    (= rhs - A x_new, cg_solver.cpp:277-298). Against the oracle, which
    recomputes the reference's way, with a recompute every 5 iterations."""
    # The count is bounded loosely: with a recompute every 5 iterations it
    # moves by up to ~15-20 % with summation order alone, fused or not (n =
    # 4096, eps = 1e-8: 61 unfused / 62 fused vs 71; n = 2048, eps = 1e-6:
    # 37 vs 43). The checks that pin the fused formula are x, the true
    # residual and the (u, alpha, beta) trace through the recompute at
    # iteration 5.
    a = oracle.generate_spd(n, b, seed=17)
    rhs = oracle.generate_rhs(n, b, seed=17)
    ref = oracle.solve_cg(n, b, a, rhs, eps=1e-6, recompute_interval=5)
    r = hs.solve_cg(hs.BlockedSPDMatrix(n, b, a), hs.BlockVector(n, b, rhs),
                    hs.SolverConfig(block_size=b, eps=1e-6, recompute_interval=5,
                                    record_trace=True), rt)
    st = r.stats
    assert st.converged and abs(st.iterations - ref["iterations"]) <= max(3, 0.2 * ref["iterations"])
    assert st.recomputations == st.iterations // 5
    assert st.true_residual <= 2e-6 * np.sqrt(st.u0)
    x = r.x.values[:n]
    assert np.linalg.norm(x - ref["x"][:n]) <= 1e-6 * np.linalg.norm(ref["x"][:n])
    tr = np.array([[t.u, t.alpha, t.beta] for t in st.trace[:6]])
    np.testing.assert_allclose(tr, ref["trace"][:6], rtol=1e-10)


@pytest.mark.parametrize("n,b,slices", [(4096, 512, 0), (4096, 512, 4), (4096, 512, 5),
                                        (2048, 128, 4), (3000, 128, 6)])
def test_mixed_precision_refined_solve_matches_oracle(oracle, n, b, slices):
    """hs_solve_spd_refine: a factor with few INT8 Ozaki slices, refined in
    FP64 against the unmodified A, reaches the requested residual and the
    oracle's solution; A is left intact; the DMMA factor needs no refinement
    step (tol above its first-solve residual)."""
    rt = hs.Runtime()
    a = oracle.generate_spd(n, b, seed=42)
    rhs = oracle.generate_rhs(n, b, seed=42)
    ref = oracle.solve_spd(n, b, a, rhs)
    m = hs.DeviceMatrix(rt, n, b).upload(a)
    work = hs.DeviceMatrix(rt, n, b)
    d_rhs = dev(rhs)
    d_x = torch.zeros_like(d_rhs)
    # refine to the FP64 floor (tol = 0: stop when a step no longer halves
    # the residual); the module's Cholesky tolerance ||b - Ax|| <= 1e-10 ||b||
    # and at least the direct FP64 solve's residual
    st = H.solve_spd_refine_device(rt, m, work, d_rhs.data_ptr(), d_x.data_ptr(),
                                   slices=slices, max_iters=20, tol=0.0)
    x = d_x.cpu().numpy()
    assert st.rel_residual <= 1e-10, st
    assert st.rel_residual <= 1.5 * ref["true_residual"] / np.linalg.norm(rhs), st
    assert np.linalg.norm(x - ref["x"]) <= 1e-8 * np.linalg.norm(ref["x"]), st
    assert st.iterations < 20, st  # stopped on the floor, not the cap
    if slices == 0:
        assert st.iterations <= 2, st  # the FP64 factor: at most a halving step or two
    elif slices <= 5:
        assert st.iterations >= 2, st
    # A is unmodified: the FP64 residual through it matches the reported one
    res = H.true_residual_device(rt, m, d_x.data_ptr(), d_rhs.data_ptr())
    assert abs(res / np.linalg.norm(rhs) - st.rel_residual) <= 1e-3 * st.rel_residual + 1e-16


def test_mixed_precision_refine_rejects_bad_arguments():
    rt = hs.Runtime()
    m = hs.DeviceMatrix(rt, 1024, 128)
    w = hs.DeviceMatrix(rt, 1024, 256)
    d = torch.zeros(1024, dtype=torch.float64, device="cuda")
    with pytest.raises(hs.ConfigError):
        H.solve_spd_refine_device(rt, m, w, d.data_ptr(), d.data_ptr(), slices=5)
    w2 = hs.DeviceMatrix(rt, 1024, 128)
    with pytest.raises(hs.ConfigError):
        H.solve_spd_refine_device(rt, m, w2, d.data_ptr(), d.data_ptr(), slices=9)


def test_mixed_precision_refine_world1_block_cyclic(oracle):
    """The refined solve through a world-1 NCCL communicator on a block-cyclic
    matrix (distributed factorization path, 1 x 1 grid)."""
    n, b = 4096, 512
    rt = hs.Runtime.distributed(0, 0, 1, hs.Runtime.nccl_unique_id())
    try:
        a = oracle.generate_spd(n, b, seed=42)
        rhs = oracle.generate_rhs(n, b, seed=42)
        ref = oracle.solve_spd(n, b, a, rhs)
        m = hs.DeviceMatrix(rt, n, b, cyclic=True).upload(a)
        work = hs.DeviceMatrix(rt, n, b, cyclic=True)
        d_rhs = dev(rhs)
        d_x = torch.zeros_like(d_rhs)
        st = H.solve_spd_refine_device(rt, m, work, d_rhs.data_ptr(), d_x.data_ptr(),
                                       slices=4, max_iters=20)
        x = d_x.cpu().numpy()
        assert st.rel_residual <= 1e-10 and st.iterations >= 2, st
        assert np.linalg.norm(x - ref["x"]) <= 1e-8 * np.linalg.norm(ref["x"]), st
    finally:
        rt.close()
