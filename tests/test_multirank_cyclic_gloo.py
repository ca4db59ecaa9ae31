"""CPU, world_size 4 (gloo, 2 x 2 grid): the 2D block-cyclic Cholesky
protocol of the multi-GPU path (hs_chol.cu potrf_run_dist).

Per column j the GPU path does: the owner of (j, j) factors it; L_jj is
broadcast; the owners of panel tiles (i, j) solve them in place; every panel
tile is broadcast from its owner into a panel buffer on every rank; every
rank updates only the trailing tiles it owns. The owner map is the product's
(hs::cyclic_owner: rank = (i mod P) * Q + (j mod Q), grid from
hs::cyclic_grid). This test restates that protocol with torch.distributed
broadcasts over gloo and checks the assembled factor against the oracle.
"""
import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

N_, B_ = 192, 16


def grid(world):
    p = 1
    d = 1
    while d * d <= world:
        if world % d == 0:
            p = d
        d += 1
    return p, world // p


def owner(i, j, P, Q):
    return (i % P) * Q + (j % Q)


def worker(rank, world, port, a_packed, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    b, N = B_, (N_ + B_ - 1) // B_
    P, Q = grid(world)
    tri = lambda i, j: i * (i + 1) // 2 + j  # noqa: E731
    full = a_packed.reshape(-1, b, b)
    mine = {(i, j): full[tri(i, j)].copy() for i in range(N) for j in range(i + 1)
            if owner(i, j, P, Q) == rank}

    def bcast(tile, root):
        t = torch.from_numpy(np.ascontiguousarray(tile) if tile is not None
                             else np.zeros((b, b)))
        dist.broadcast(t, root)
        return t.numpy()

    for j in range(N):
        dj = owner(j, j, P, Q)
        if dj == rank:
            d = np.tril(mine[(j, j)])
            L = np.linalg.cholesky(d + np.tril(d, -1).T)
            mine[(j, j)] = L  # lower part is L; the upper half is stale
        Ljj = bcast(mine.get((j, j)) if dj == rank else None, dj)
        Ljj = np.tril(Ljj)
        for i in range(j + 1, N):  # panel TRSM on owned tiles: X L^T = A
            if (i, j) in mine:
                mine[(i, j)] = np.linalg.solve(Ljj, mine[(i, j)].T).T
        panel = {}
        for i in range(j + 1, N):
            o = owner(i, j, P, Q)
            panel[i] = bcast(mine.get((i, j)) if o == rank else None, o)
        for i in range(j + 1, N):  # trailing update of owned tiles
            for k in range(j + 1, i + 1):
                if (i, k) in mine:
                    upd = panel[i] @ panel[k].T
                    if i == k:
                        mine[(i, k)] = mine[(i, k)] - np.tril(upd)
                    else:
                        mine[(i, k)] = mine[(i, k)] - upd
    out[rank] = {k: v for k, v in mine.items()}
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_block_cyclic_cholesky_protocol_matches_oracle(oracle):
    n, b = N_, B_
    N = (n + b - 1) // b
    a = oracle.generate_spd(n, b, seed=42)
    st, L_ref, _, _ = oracle.factorize(n, b, a)
    assert st == 0
    world = 4
    with mp.Manager() as mgr:
        out = mgr.dict()
        mp.spawn(worker, args=(world, _free_port(), a, out), nprocs=world, join=True)
        parts = {r: dict(out[r]) for r in range(world)}
    P, Q = grid(world)
    assert (P, Q) == (2, 2)
    got = np.zeros_like(L_ref).reshape(-1, b, b)
    seen = 0
    for r, tiles in parts.items():
        for (i, j), t in tiles.items():
            assert owner(i, j, P, Q) == r
            got[i * (i + 1) // 2 + j] = t
            seen += 1
    assert seen == N * (N + 1) // 2
    ref = L_ref.reshape(-1, b, b)
    for i in range(N):
        for j in range(i + 1):
            g, r_ = got[i * (i + 1) // 2 + j], ref[i * (i + 1) // 2 + j]
            if i == j:
                g, r_ = np.tril(g), np.tril(r_)
            assert np.abs(g - r_).max() <= 1e-10 * np.abs(a).max()


def test_cyclic_grid_matches_product():
    # the grid used here is the product's hs::cyclic_grid rule
    assert [grid(w) for w in (1, 2, 4, 8, 6)] == [(1, 1), (1, 2), (2, 2), (2, 4), (2, 3)]
