"""CPU: pin the oracle (oracle/hs_oracle.c) to the reference.

1. Against the golden fixtures generated from the REAL reference
   (tests/golden/make_golden.py) — runs anywhere, bitwise.
2. Against oracle/_ref (the reference compiled from /root/reference) when it
   is present — bitwise, over more shapes.
3. The reference's own known-answer tests (test_block_kernels.cpp etc.).
"""
import hashlib
import json
import os

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = np.load(os.path.join(HERE, "golden", "reference_golden.npz"))
META = json.load(open(os.path.join(HERE, "golden", "reference_golden.json")))


def digest(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype="<f8").tobytes()).hexdigest()


# ---------------------------------------------------------------------------
# 1. golden fixtures (bitwise)


def test_golden_assembly_and_symv(oracle):
    a = oracle.generate_spd(45, 8, seed=17)
    assert np.array_equal(a, GOLD["spd_45_8_s17"])
    x = oracle.generate_rhs(45, 8, seed=10)
    assert np.array_equal(x, GOLD["rhs_45_8_s10"])
    assert np.array_equal(oracle.symv(45, 8, a, x), GOLD["symv_45_8"])
    assert np.array_equal(oracle.generate_inputs(100, 2, 42), GOLD["inputs_100_2_s42"])


def test_golden_cfg1_cg_and_cholesky(oracle):
    n, b = 1024, 128
    a = oracle.generate_spd(n, b, seed=42)
    assert digest(a) == META["cfg1_spd_sha256"]
    rhs = oracle.generate_rhs(n, b, seed=42)
    assert np.array_equal(rhs, GOLD["cfg1_rhs"])
    cg = oracle.solve_cg(n, b, a, rhs, eps=1e-6, max_iters=500, recompute_interval=50)
    assert cg["iterations"] == META["cfg1_cg"]["iterations"] == 30
    assert cg["u0"] == META["cfg1_cg"]["u0"]
    assert cg["true_residual"] == META["cfg1_cg"]["true_residual"]
    assert np.array_equal(cg["x"], GOLD["cfg1_cg_x"])
    assert np.array_equal(cg["trace"], GOLD["cfg1_cg_trace"])
    sp = oracle.solve_spd(n, b, a, rhs)
    assert sp["status"] == 0
    assert digest(sp["L"]) == META["cfg1_L_sha256"]
    assert np.array_equal(sp["x"], GOLD["cfg1_spd_x"])
    assert sp["true_residual"] == META["cfg1_spd_true_residual"]


def test_golden_small_factor_and_split_cg(oracle):
    a = oracle.generate_spd(128, 16, seed=5)
    st, L, _, _ = oracle.factorize(128, 16, a)
    assert st == 0 and np.array_equal(L, GOLD["chol_128_16_L"])
    # the reference's fraction=0.5 split gives the homogeneous result bitwise
    # (test_cg_solver.cpp:93-129); the oracle is homogeneous
    a99 = oracle.generate_spd(128, 16, seed=99)
    cg = oracle.solve_cg(128, 16, a99, oracle.generate_rhs(128, 16, 99), eps=1e-9,
                         max_iters=300)
    assert np.array_equal(cg["x"], GOLD["cg_128_16_s99_x"])
    assert np.array_equal(cg["trace"], GOLD["cg_128_16_s99_trace"])


# ---------------------------------------------------------------------------
# 2. against the compiled reference (dev container)


@pytest.mark.parametrize("n,b,seed", [(8, 2, 77), (64, 16, 3), (100, 16, 5), (1000, 64, 1),
                                      (333, 7, 9), (512, 128, 4)])
def test_oracle_bitwise_vs_reference(oracle, reference, n, b, seed):
    a = oracle.generate_spd(n, b, seed=seed)
    assert np.array_equal(a, reference.generate_spd(n, b, seed=seed))
    rhs = oracle.generate_rhs(n, b, seed)
    assert np.array_equal(rhs, reference.generate_rhs(n, b, seed))
    assert np.array_equal(oracle.symv(n, b, a, rhs), reference.symv(n, b, a, rhs))
    c1 = oracle.solve_cg(n, b, a, rhs, eps=1e-8, max_iters=300, recompute_interval=7)
    c2 = reference.solve_cg(n, b, a, rhs, eps=1e-8, max_iters=300, recompute_interval=7,
                            workers=3)
    assert c1["iterations"] == c2["iterations"]
    assert c1["recomputations"] == c2["recomputations"]
    assert np.array_equal(c1["x"], c2["x"]) and np.array_equal(c1["trace"], c2["trace"])
    assert c1["true_residual"] == c2["true_residual"]
    st, L, _, _ = oracle.factorize(n, b, a)
    r = reference.factorize(n, b, a)
    assert st == r["status"] == 0 and np.array_equal(L, r["L"])
    s1, s2 = oracle.solve_spd(n, b, a, rhs), reference.solve_spd(n, b, a, rhs)
    assert np.array_equal(s1["x"], s2["x"])
    assert s1["true_residual"] == s2["true_residual"]


def test_oracle_not_spd_matches_reference(oracle, reference):
    a = oracle.generate_spd(64, 16, seed=2)
    # element (40, 40): tile (2, 2), row/col 8
    k = (2 * 3 // 2 + 2) * 256 + 8 * 16 + 8
    a[k] = -5.0
    st, _, row, piv = oracle.factorize(64, 16, a)
    r = reference.factorize(64, 16, a)
    assert st == r["status"] == 2
    assert (row, piv) == (r["block_row"], r["pivot"]) == (2, 8)


def test_partition_matches_reference(oracle, reference):
    for rows in (1, 4, 7, 64):
        for f in (0.0, 0.1, 0.25, 0.5, 0.85, 1.0):
            assert oracle.partition_for_fraction(f, rows) == \
                reference.lib.ref_partition_for_fraction(f, rows)
            for col in range(rows):
                assert oracle.cholesky_border(f, col, rows) == \
                    reference.lib.ref_cholesky_border(f, col, rows)


# ---------------------------------------------------------------------------
# 3. the reference's known-answer tests, on the oracle


def test_kat_potf_block(oracle):
    # test_block_kernels.cpp:33-55
    d = np.array([4.0, 2.0, 2.0, 3.0])
    assert oracle.lib.hso_potf_block(d, 2, None) == 0
    assert d[0] == 2.0 and d[2] == 1.0 and abs(d[3] - np.sqrt(2)) <= 1e-15 and d[1] == 2.0
    bad = np.array([1.0, 2.0, 2.0, 1.0])
    import ctypes
    piv = ctypes.c_int64(-1)
    assert oracle.lib.hso_potf_block(bad, 2, ctypes.byref(piv)) == 2 and piv.value == 1


def test_kat_trsm_gemm_syrk(oracle):
    s2 = np.sqrt(2.0)
    x = np.array([2.0, 0.0, 0.0, 2.0])
    assert oracle.lib.hso_trsm_block(x, np.array([2.0, 0.0, 1.0, s2]), 2, None) == 0
    assert np.allclose(x, [1.0, -s2 / 2, 0.0, s2], rtol=1e-15, atol=1e-15)
    c = np.array([1.0, 0.0, 0.0, 1.0])
    oracle.lib.hso_gemm_update(c, np.array([1.0, 2.0, 3.0, 4.0]), np.array([1.0, 0, 0, 1.0]), 2)
    assert c.tolist() == [0.0, -2.0, -3.0, -3.0]
    c = np.array([5.0, 42.0, 2.0, 5.0])
    oracle.lib.hso_syrk_update(c, np.ones(4), 2)
    assert c.tolist() == [3.0, 42.0, 0.0, 3.0]


def test_kat_dot_and_cg_identity(oracle):
    u = np.array([1.0, 2.0, 3.0])
    v = np.array([4.0, 5.0, 6.0])
    assert oracle.dot(3, 1, u, v) == 32.0
    n, b = 64, 16
    ident = np.zeros(10 * 256)
    for i in range(4):
        k = i * (i + 1) // 2 + i
        ident[k * 256:(k + 1) * 256] = np.eye(16).ravel()
    rhs = oracle.generate_rhs(n, b, 1)
    cg = oracle.solve_cg(n, b, ident, rhs)
    assert cg["iterations"] == 1 and cg["converged"] and np.array_equal(cg["x"], rhs)
