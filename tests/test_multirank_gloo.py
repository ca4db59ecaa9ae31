"""CPU, world_size 2 (gloo): the row-sharded CG protocol of the multi-GPU path.

The GPU path (hs_cg.cu cg_run, world > 1) shards the packed tiles by block
rows with the product's own partition (hs_partition_rows), keeps vectors in a
padded rank-chunk layout whose chunks end in 2 * world doubles of dot slots,
and per iteration does
  1. local packed SYMV -> full-length partial t (own rows + transposed
     contributions to earlier rows), and this rank's s^T t_partial as a
     double-double written into slot `rank` of every chunk,
  2. reduce-scatter of the partial -> own rows of t and, in the slots, every
     rank's s^T t partial (exact: the other ranks' slots are 0); rank-order
     combine -> alpha, identical on every rank,
  3. local x / r updates and r^T r partial into slot `rank` of the r chunk,
  4. all-gather of the r chunks (rows + slots); rank-order combine -> beta;
     s = r + beta s on the full vector by every rank,
  5. on recompute iterations, also an all-gather of x.
Two collectives per iteration. This test restates exactly that protocol with
torch.distributed over gloo (NCCL needs GPUs; gloo has no reduce-scatter, so
all-reduce + slice stands in) and checks the solution against the
single-process oracle CG.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

N_, B_ = 512, 32


def two_sum(a, b):
    s = a + b
    bb = s - a
    return s, (a - (s - bb)) + (b - bb)


def dd_add(x, y):
    s, e = two_sum(x[0], y[0])
    lo = e + (x[1] + y[1])
    hi = s + lo
    return hi, lo - (hi - s)


def dd_sum(vals):
    acc = (0.0, 0.0)
    for v in vals:
        acc = dd_add(acc, (float(v), 0.0))
    return acc


def local_symv(tiles, lo, hi, b, s_full_std, nrows):
    """Contributions of block rows [lo, hi) (packed tiles) to the full t."""
    t = np.zeros(nrows * b)
    k = 0
    for i in range(lo, hi):
        for j in range(i + 1):
            blk = tiles[k].reshape(b, b)
            k += 1
            sj = s_full_std[j * b:(j + 1) * b]
            si = s_full_std[i * b:(i + 1) * b]
            if i == j:
                lower = np.tril(blk)
                t[i * b:(i + 1) * b] += lower @ sj + np.tril(blk, -1).T @ si
            else:
                t[i * b:(i + 1) * b] += blk @ sj
                t[j * b:(j + 1) * b] += blk.T @ si
    return t


def worker(rank, world, port, a_packed, rhs, bounds, iters, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    b, N = B_, (N_ + B_ - 1) // B_
    lo, hi = bounds[rank], bounds[rank + 1]
    lmax = max(bounds[g + 1] - bounds[g] for g in range(world))
    rows_len = lmax * b
    chunk = rows_len + 2 * world  # rows, then one (hi, lo) slot per rank
    tri = lambda i: i * (i + 1) // 2  # noqa: E731
    tiles = a_packed.reshape(-1, b * b)[tri(lo):tri(hi)]

    def to_padded(v_std):
        out = np.zeros(world * chunk)
        for g in range(world):
            r0, r1 = bounds[g], bounds[g + 1]
            out[g * chunk:g * chunk + (r1 - r0) * b] = v_std[r0 * b:r1 * b]
        return out

    def to_std(v_pad):
        out = np.zeros(N * b)
        for g in range(world):
            r0, r1 = bounds[g], bounds[g + 1]
            out[r0 * b:r1 * b] = v_pad[g * chunk:g * chunk + (r1 - r0) * b]
        return out

    def allgather_chunk(local):
        parts = [torch.zeros(chunk, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(parts, torch.from_numpy(local.copy()))
        return np.concatenate([p.numpy() for p in parts])

    def reduce_scatter(full_pad):
        t = torch.from_numpy(full_pad.copy())
        dist.all_reduce(t)
        return t.numpy()[rank * chunk:(rank + 1) * chunk].copy()

    def dd_dot(u, v, nblk):
        return dd_sum([u[i * b:(i + 1) * b] @ v[i * b:(i + 1) * b] for i in range(nblk)])

    def combine(slots):
        acc = tuple(slots[0])
        for p in slots[1:]:
            acc = dd_add(acc, tuple(p))
        return acc[0] + acc[1]

    def setup_dot(u, v):  # u0 (and the exit residual): a scalar all-gather
        part = dd_dot(u, v, hi - lo)
        parts = [torch.zeros(2, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(parts, torch.tensor(part, dtype=torch.float64))
        return combine([p.tolist() for p in parts])

    own = (hi - lo) * b
    rhs_loc = np.zeros(chunk)
    rhs_loc[:own] = rhs[lo * b:hi * b]
    x = np.zeros(chunk)
    r = rhs_loc.copy()
    s_full = allgather_chunk(rhs_loc)
    u = setup_dot(rhs_loc, rhs_loc)
    limit = 1e-12 * u  # eps = 1e-6, as cg_solver.cpp:248
    done = 0
    for it in range(1, iters + 1):
        t_std = local_symv(tiles, lo, hi, b, to_std(s_full), N)
        t_part = to_padded(t_std)
        # s^T t_partial over the full length, into slot `rank` of every chunk
        part = dd_sum([to_std(s_full)[i * b:(i + 1) * b] @ t_std[i * b:(i + 1) * b]
                       for i in range(N)])
        for g in range(world):
            t_part[g * chunk + rows_len + 2 * rank:g * chunk + rows_len + 2 * rank + 2] = part
        t = reduce_scatter(t_part)
        alpha = u / combine([t[rows_len + 2 * g:rows_len + 2 * g + 2] for g in range(world)])
        s_loc = s_full[rank * chunk:(rank + 1) * chunk]
        x[:rows_len] = x[:rows_len] + alpha * s_loc[:rows_len]
        if it % 50 == 0:
            x_full = allgather_chunk(x)
            t = reduce_scatter(to_padded(local_symv(tiles, lo, hi, b, to_std(x_full), N)))
            r[:rows_len] = rhs_loc[:rows_len] - t[:rows_len]
        else:
            r[:rows_len] = r[:rows_len] - alpha * t[:rows_len]
        r[rows_len + 2 * rank:rows_len + 2 * rank + 2] = dd_dot(r, r, hi - lo)
        r_full = allgather_chunk(r)
        unew = combine([r_full[g * chunk + rows_len + 2 * g:g * chunk + rows_len + 2 * g + 2]
                        for g in range(world)])
        beta = unew / u
        u = unew
        s_full = r_full + beta * s_full  # every rank, full length
        done = it
        if u <= limit:
            break
    x_full = to_std(allgather_chunk(x))
    out[rank] = (x_full, u, done)
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_row_sharded_cg_protocol_matches_oracle(oracle):
    import paper_2605_13209_b200 as hs
    n, b = N_, B_
    N = (n + b - 1) // b
    a = oracle.generate_spd(n, b, seed=42)
    rhs = oracle.generate_rhs(n, b, seed=42)
    bounds = hs.partition_rows(N, 2)
    assert bounds[0] == 0 and bounds[-1] == N and 0 < bounds[1] < N
    iters = 500
    ref = oracle.solve_cg(n, b, a, rhs, eps=1e-6, max_iters=iters)
    with mp.Manager() as mgr:
        out = mgr.dict()
        mp.spawn(worker, args=(2, _free_port(), a, rhs, bounds, iters, out), nprocs=2,
                 join=True)
        x0, u0, k0 = out[0]
        x1, u1, k1 = out[1]
    # every rank ends with the same full solution, scalars and iteration count
    assert np.array_equal(x0, x1) and u0 == u1 and k0 == k1
    # the GPU-vs-oracle CG tolerance (tests/test_gpu_parity.py)
    assert abs(k0 - ref["iterations"]) <= 2
    assert np.linalg.norm(x0 - ref["x"]) <= 1e-6 * np.linalg.norm(ref["x"])


@pytest.mark.parametrize("rows,world", [(256, 2), (1024, 8), (5, 2)])
def test_padded_layout_roundtrip(rows, world):
    import paper_2605_13209_b200 as hs
    bounds = hs.partition_rows(rows, world)
    lmax = max(bounds[g + 1] - bounds[g] for g in range(world))
    seen = set()
    for g in range(world):
        for i in range(bounds[g], bounds[g + 1]):
            off = g * lmax + (i - bounds[g])
            assert off not in seen
            seen.add(off)
    assert len(seen) == rows
