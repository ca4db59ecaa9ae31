"""Row K9: the factor's non-finite scan (cholesky_solver.cpp:222-238).

A +Inf on the diagonal of A passes every pivot test of potf_block
(block_kernels.cpp:9-21: sqrt(+Inf) > 0), turns the column below it into
exact zeros (finite / Inf) and leaves L(p, p) = +Inf, so the reference ends
in check_finite -> NumericalError("factor has a non-finite value in block
(i, i)") instead of NotSpdError. The GPU must give the same outcome on every
factorization engine: FP64 DMMA (b = 128 / 512), INT8-emulated FP64, the
small-b SIMT path, and the 2D block-cyclic (world-1 NCCL) path — checked
against oracle/_ref where it travelled with the repo, else the C
restatement.
"""
import numpy as np
import pytest

import paper_2605_13209_b200 as hs
from paper_2605_13209_b200 import hsolve as H

pytestmark = pytest.mark.gpu

CASES = [(64, 16, 40), (1024, 128, 657), (1024, 128, 3), (2048, 512, 700), (2048, 512, 2047)]


def _inf_diag(values, n, b, p):
    a = hs.BlockedSPDMatrix(n, b, values.copy())
    a.set(p, p, np.inf)
    return a


def _expected(reference_or_oracle, n, b, a):
    """Status code from the CPU reference."""
    from oracle import Reference
    r = reference_or_oracle
    if isinstance(r, Reference):
        return r.factorize(n, b, a.values)["status"]
    st, _, _, _ = r.factorize(n, b, a.values)
    return st


@pytest.fixture(scope="module")
def cpu_ref():
    from oracle import Oracle, Reference
    return Reference() if Reference.available() else Oracle()


@pytest.mark.parametrize("n,b,p", CASES)
@pytest.mark.parametrize("slices", [0, 8], ids=["dmma", "int8_emulated"])
def test_inf_diagonal_numerical_error(rt, oracle, cpu_ref, n, b, p, slices):
    if slices and b % 128:
        pytest.skip("the INT8 engine serves b % 128 == 0")
    a = _inf_diag(oracle.generate_spd(n, b, seed=4), n, b, p)
    assert _expected(cpu_ref, n, b, a) == 1 + 3  # ErrorKind::numerical
    rt.set_cholesky_gemm(slices)
    try:
        with pytest.raises(hs.NumericalError) as ei:
            hs.factorize(a, hs.SolverConfig(block_size=b), rt)
    finally:
        rt.set_cholesky_gemm(0)
    i = p // b
    assert f"block ({i}, {i})" in str(ei.value)
    # solve_spd surfaces the same error (cholesky_solver.cpp:286)
    a2 = _inf_diag(oracle.generate_spd(n, b, seed=4), n, b, p)
    with pytest.raises(hs.NumericalError):
        hs.solve_spd(a2, hs.generate_rhs(n, b, 4), hs.SolverConfig(block_size=b), rt)


@pytest.mark.parametrize("n,b,p", [(1024, 128, 657), (2048, 512, 700)])
@pytest.mark.parametrize("slices", [0, 8], ids=["dmma", "int8_emulated"])
def test_inf_diagonal_numerical_error_block_cyclic(oracle, n, b, p, slices):
    rt = hs.Runtime.distributed(0, 0, 1, hs.Runtime.nccl_unique_id())
    try:
        a = _inf_diag(oracle.generate_spd(n, b, seed=4), n, b, p)
        m = hs.DeviceMatrix(rt, n, b, cyclic=True).upload(a)
        rt.set_cholesky_gemm(slices)
        with pytest.raises(hs.NumericalError) as ei:
            H.potrf_device(rt, m)
        i = p // b
        assert f"block ({i}, {i})" in str(ei.value)
        m.free()
    finally:
        rt.close()


def test_nan_stays_not_spd(rt, oracle, cpu_ref):
    """A NaN fails the pivot test first (NotSpdError, as the reference)."""
    n, b, p = 1024, 128, 300
    a = hs.BlockedSPDMatrix(n, b, oracle.generate_spd(n, b, seed=4))
    a.set(p, p, np.nan)
    assert _expected(cpu_ref, n, b, a) == 1 + 1  # ErrorKind::not_spd
    with pytest.raises(hs.NotSpdError) as ei:
        hs.factorize(a, hs.SolverConfig(block_size=b), rt)
    assert ei.value.block_row == p // b and ei.value.pivot_index == p % b
