"""CPU: the C-ABI library loads, exports every symbol include/hs_cuda.h
declares, and its host-only entry points (no GPU needed) agree with the oracle
bitwise: RNG, points, median length scale, rhs, work split."""
import ctypes as C
import os
import re

import numpy as np
import pytest

import paper_2605_13209_b200 as hs
from paper_2605_13209_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "hs_cuda.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(hs_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    L = _lib.lib()
    decl = declared_symbols()
    assert len(decl) >= 40
    missing = [s for s in decl if not hasattr(L, s)]
    assert not missing, missing
    assert sorted(_lib.EXPORTED) == decl


def test_host_shim_exports_reference_api():
    so = os.path.join(ROOT, "paper_2605_13209_b200", "libhsolve_b200.so")
    if not os.path.exists(so):
        pytest.skip("C++ shim not built")
    out = os.popen(f"nm -DC --defined-only {so}").read()
    for sym in ["hsolve::solve_cg(", "hsolve::factorize(", "hsolve::solve_spd(",
                "hsolve::forward_substitute(", "hsolve::back_substitute(",
                "hsolve::generate_spd(", "hsolve::generate_rhs(",
                "hsolve::partition_for_fraction(", "hsolve::cholesky_border(",
                "hsolve::BlockedSPDMatrix::BlockedSPDMatrix("]:
        assert sym in out, sym


def test_rng_and_points_match_oracle(oracle):
    L = _lib.lib()
    for key, ctr in [(0, 0), (42 ^ 0x7268730000000001, 17), (2**63 + 5, 2**40)]:
        assert L.hs_rng_at(key, ctr) == oracle.lib.hso_rng_at(key, ctr)
        assert L.hs_rng_uniform_pm1(key, ctr) == oracle.lib.hso_uniform_pm1(key, ctr)
    for n, dim, seed in [(1, 3, 7), (100, 2, 42), (1000, 4, 5)]:
        p = hs.generate_inputs(n, dim, seed)
        assert np.array_equal(p, oracle.generate_inputs(n, dim, seed))
        assert hs.median_pairwise_distance(p, n, dim) == \
            oracle.median_pairwise_distance(p, n, dim)


@pytest.mark.parametrize("n,b,seed", [(45, 8, 10), (1024, 128, 42), (33, 8, 9), (5, 7, 1)])
def test_rhs_matches_oracle(oracle, n, b, seed):
    assert np.array_equal(hs.generate_rhs(n, b, seed).values, oracle.generate_rhs(n, b, seed))


def test_partition_matches_oracle(oracle):
    for rows in (1, 4, 7, 64):
        for f in (0.0, 0.1, 0.25, 0.5, 0.85, 1.0):
            assert hs.partition_for_fraction(f, rows).split_row == \
                oracle.partition_for_fraction(f, rows)
            for col in range(rows):
                assert hs.cholesky_border(f, col, rows) == oracle.cholesky_border(f, col, rows)
    with pytest.raises(hs.ConfigError):
        hs.partition_for_fraction(1.5, 4)
    with pytest.raises(hs.ConfigError):
        hs.partition_for_fraction(0.5, 0)


@pytest.mark.parametrize("rows,world", [(256, 1), (256, 2), (1024, 8), (7, 4), (3, 8), (64, 3)])
def test_partition_rows_balances_tiles(rows, world):
    b = hs.partition_rows(rows, world)
    assert b[0] == 0 and b[-1] == rows and all(x <= y for x, y in zip(b, b[1:]))
    tiles = [(hi * (hi + 1) - lo * (lo + 1)) // 2 for lo, hi in zip(b, b[1:])]
    T = rows * (rows + 1) // 2
    if rows >= 4 * world:
        # every rank within one block row of its share
        assert max(tiles) - T / world <= rows


def test_config_validation_mirrors_reference():
    # solver_config.cpp:9-26
    for bad in [dict(eps=0.0), dict(fraction=1.5), dict(block_size=0), dict(workers_a=0),
                dict(slowdown_b=0.5), dict(gpus=0)]:
        with pytest.raises(hs.ConfigError):
            hs.SolverConfig(**bad).validate()
    hs.SolverConfig().validate()


def test_host_storage_semantics():
    # blocked_matrix.cpp:8-82, test_core_types.cpp
    m = hs.BlockedSPDMatrix(10, 4)
    assert m.rows == 3 and m.block_count == 6 and m.padded_n == 12
    assert m.block(2, 2)[2, 2] == 1.0 and m.block(2, 2)[3, 3] == 1.0  # identity padding
    m.set(1, 8, 3.5)
    assert m.element(8, 1) == 3.5 and m.element(1, 8) == 3.5
    assert hs.block_index(3, 2, 4) == 8
    with pytest.raises(IndexError):
        hs.block_index(2, 3, 4)
    v = hs.BlockVector(10, 4)
    assert v.padded_n == 12 and np.all(v.values == 0.0)
    with pytest.raises(hs.ConfigError):
        hs.BlockedSPDMatrix(0, 4)


def test_no_gpu_means_loud_failure():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(hs.DeviceError):
        hs.Runtime()


def test_refine_solve_rejects_null_arguments_without_a_gpu():
    # hs_solve_spd_refine validates its arguments before touching a device
    L = _lib.lib()
    st = _lib.RefineStats()
    r = L.hs_solve_spd_refine(None, None, None, None, None, 4, 10, 0.0, C.byref(st))
    assert r == 1  # HS_ERR_CONFIG
    assert b"null pointer" in L.hs_last_error()
