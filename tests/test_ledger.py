"""Communication ledger (transfer_ledger.hpp:9-52): every NCCL collective a
multi-rank context issues is logged with its kind, payload bytes and step.
The closed-form per-iteration / per-column contracts below play the role of
the reference's ledger tests (test_cg_solver.cpp:131-187,
test_cholesky_solver.cpp:125-176) for the G-GPU protocols:

* CG, iteration k: 2 subvector entries and no scalar one: the reduce-scatter
  of t carries every rank's s^T t partial, the all-gather of r every rank's
  r^T r partial (2 doubles per rank appended to each rank chunk), so the
  two dot reductions of the reference's iteration cost no collective of
  their own; plus 2 more subvector entries on each recompute iteration
  (all-gather of x, reduce-scatter of A x); setup and exit entries carry
  step -1 (one scalar all-gather each for u0 and the residual); the result
  all-gather is one `result` entry.
* Cholesky, column j: 2 + (N - j - 1) block entries (L_jj, its inverse
  blocks, and one broadcast per panel tile), then one scalar status
  all-reduce at step -1.
* Single-GPU contexts issue no collectives: empty ledger (the reference's
  homogeneous runs, test_cg_solver.cpp:178-187).

Run on one GPU through a world-size-1 communicator (same call sequence as
any world size; bytes are those of a world-1 chunk).
"""
from collections import Counter

import numpy as np
import pytest
import torch

import paper_2605_13209_b200 as hs
from paper_2605_13209_b200 import hsolve as H

pytestmark = pytest.mark.gpu


def by_step(entries, kind):
    c = Counter()
    for e in entries:
        if e.kind == kind:
            c[e.step] += 1
    return c


@pytest.mark.parametrize("iters,interval,recomputes", [(7, 0, 0), (12, 5, 2)])
def test_cg_ledger_contract(iters, interval, recomputes):
    n, b = 1024, 128
    rt = hs.Runtime.distributed(0, 0, 1, hs.Runtime.nccl_unique_id())
    try:
        m = hs.generate_spd_device(rt, n, b, seed=21)
        rhs = torch.from_numpy(hs.generate_rhs(n, b, 21).values).cuda()
        x = torch.zeros_like(rhs)
        rt.ledger(clear=True)
        st = hs.solve_cg_device(rt, m, rhs.data_ptr(), x.data_ptr(),
                                hs.SolverConfig(block_size=b, eps=1e-300, max_iters=iters,
                                                recompute_interval=interval))
        assert st.iterations == iters and st.recomputations == recomputes
        led = rt.ledger()
        assert all(e.direction == "bidirectional" for e in led)
        sc, sv = by_step(led, "scalar"), by_step(led, "subvector")
        rec_steps = {k for k in range(1, iters + 1) if interval and k % interval == 0}
        for k in range(1, iters + 1):
            assert sc[k] == 0, k
            assert sv[k] == 2 + (2 if k in rec_steps else 0), k
        assert sum(v for s, v in sc.items() if s >= 1) == 0
        assert sum(v for s, v in sv.items() if s >= 1) == 2 * iters + 2 * recomputes
        assert Counter(e.kind for e in led if e.step == -1) == {
            "scalar": 2, "subvector": 2, "result": 1}
        # world 1: the chunk is the whole vector + one (hi, lo) dot slot
        vec_bytes = (n + 2) * 8
        for e in led:
            if e.kind in ("subvector", "result"):
                assert e.bytes == vec_bytes
            elif e.kind == "scalar":
                assert e.bytes == 16  # one (hi, lo) double-double per rank
        # a second solve appends; clearing empties
        hs.solve_cg_device(rt, m, rhs.data_ptr(), x.data_ptr(),
                           hs.SolverConfig(block_size=b, eps=1e-300, max_iters=2))
        assert len(rt.ledger()) > len(led)
        rt.ledger(clear=True)
        assert rt.ledger() == []
    finally:
        rt.close()


@pytest.mark.parametrize("n,b", [(1024, 128), (2048, 512)])
def test_cholesky_ledger_contract(n, b):
    N = (n + b - 1) // b
    rt = hs.Runtime.distributed(0, 0, 1, hs.Runtime.nccl_unique_id())
    try:
        m = hs.generate_spd_device(rt, n, b, seed=3, cyclic=True)
        rt.ledger(clear=True)
        H.potrf_device(rt, m)
        led = rt.ledger()
        blk = by_step(led, "block")
        for j in range(N):
            assert blk[j] == 2 + (N - j - 1), j
        assert sum(blk.values()) == 2 * N + N * (N - 1) // 2
        f = b // 128
        sizes = Counter(e.bytes for e in led if e.kind == "block")
        tiles = N + N * (N - 1) // 2  # L_jj + panel tiles, b*b doubles each
        inv = f * 128 * 128 * 8       # the f 128x128 inverse blocks of L_jj
        if inv == b * b * 8:
            assert sizes == {inv: tiles + N}
        else:
            assert sizes == {b * b * 8: tiles, inv: N}
        assert [e.kind for e in led if e.step == -1] == ["scalar"]
        assert not any(e.kind in ("subvector", "block_row") for e in led)
    finally:
        rt.close()


def test_single_gpu_runs_log_nothing(rt):
    n, b = 512, 64
    m = hs.generate_spd_device(rt, n, b, seed=1)
    rhs = torch.from_numpy(hs.generate_rhs(n, b, 1).values).cuda()
    x = torch.zeros_like(rhs)
    hs.solve_cg_device(rt, m, rhs.data_ptr(), x.data_ptr(), hs.SolverConfig(block_size=b))
    H.potrf_device(rt, m)
    assert rt.ledger() == []
    a = hs.generate_spd(256, 32, seed=2)
    r = hs.Runtime()
    hs.solve_cg(a, hs.generate_rhs(256, 32, 2), hs.SolverConfig(block_size=32), r)
    assert r.ledger() == []
    r.close()
    np.testing.assert_equal(len(hs.Runtime().ledger()), 0)
