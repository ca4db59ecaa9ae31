"""The world > 1 code paths of the CUDA library, run on ONE GPU.

NCCL refuses two ranks on the same device, so these tests give each spawned
process (rank) a context from hs_ctx_create_custom_comm whose collectives go
through a host transport (device -> host, torch.distributed gloo, host ->
device). Everything else is the production multi-rank path: row-sharded CG
(per-rank tiles and SYMV, reduce-scatter of t, all-gather of s, rank-ordered
double-double dots, padded rank-chunk vectors) and the 2D block-cyclic
Cholesky (owned tiles, broadcasts of L_jj / inverses / panel tiles, owned
trailing pairs, status all-reduce), DMMA and INT8-emulated. Results are
compared with the oracle at the same tolerances as the single-GPU tests.
"""
import ctypes as C
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

_CUDART = None


def cudart():
    global _CUDART
    if _CUDART is None:
        for path in ("libcudart.so.12", "/usr/local/cuda/lib64/libcudart.so.12"):
            try:
                _CUDART = C.CDLL(path)
                break
            except OSError:
                continue
        _CUDART.cudaMemcpy.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_int]
    return _CUDART


def d2h(ptr, count, dtype=np.float64):
    out = np.empty(count, dtype=dtype)
    assert cudart().cudaMemcpy(out.ctypes.data, ptr, out.nbytes, 2) == 0
    return out


def h2d(ptr, arr):
    arr = np.ascontiguousarray(arr)
    assert cudart().cudaMemcpy(ptr, arr.ctypes.data, arr.nbytes, 1) == 0
    # a pageable-memory cudaMemcpy may return before the DMA lands, and the
    # library's streams are non-blocking: finish it before handing back
    assert cudart().cudaDeviceSynchronize() == 0


class GlooTransport:
    """hs_comm_ops over torch.distributed (gloo) with host staging."""

    def __init__(self, rank, world):
        self.rank, self.world = rank, world

    def allgather(self, send, recv, count):
        mine = torch.from_numpy(d2h(send, count))
        parts = [torch.empty(count, dtype=torch.float64) for _ in range(self.world)]
        dist.all_gather(parts, mine)
        h2d(recv, torch.cat(parts).numpy())

    def reduce_scatter(self, send, recv, count):
        full = torch.from_numpy(d2h(send, count * self.world))
        dist.all_reduce(full)  # gloo has no reduce_scatter: sum, keep my chunk
        h2d(recv, full[self.rank * count:(self.rank + 1) * count].numpy())

    def broadcast(self, send, recv, count, root):
        t = torch.from_numpy(d2h(send, count)) if self.rank == root else \
            torch.empty(count, dtype=torch.float64)
        dist.broadcast(t, src=root)
        h2d(recv, t.numpy())

    def allreduce_max_i64(self, buf, count):
        t = torch.from_numpy(d2h(buf, count, np.int64))
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        h2d(buf, t.numpy())


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, job, result_q):
    try:
        _work(rank, world, port, job, result_q)
    except BaseException:
        import traceback
        result_q.put((rank, {"error": traceback.format_exc()}))
        raise


def _work(rank, world, port, job, result_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys
        sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        import paper_2605_13209_b200 as hs
        from paper_2605_13209_b200 import hsolve as H
        from oracle import Oracle
        torch.cuda.set_device(0)
        rt = hs.Runtime.custom_comm(0, rank, world, GlooTransport(rank, world))
        o = Oracle()
        kind, n, b, extra = job
        a = o.generate_spd(n, b, seed=42)
        if kind == "cg":
            rhs = o.generate_rhs(n, b, seed=42)
            m = hs.DeviceMatrix(rt, n, b).upload(a)
            d_rhs = torch.from_numpy(rhs).cuda()
            d_x = torch.zeros_like(d_rhs)
            cfg = hs.SolverConfig(block_size=b, eps=extra.get("eps", 1e-6),
                                  max_iters=extra.get("max_iters", 500),
                                  recompute_interval=extra.get("recompute", 50))
            st = hs.solve_cg_device(rt, m, d_rhs.data_ptr(), d_x.data_ptr(), cfg)
            led = [(e.kind, e.step) for e in rt.ledger()]
            out = {"x": d_x.cpu().numpy(), "iters": st.iterations, "conv": st.converged,
                   "res": st.true_residual, "u0": st.u0, "ledger": led}
        elif kind == "io":
            # every rank streams its own tiles from the file, then writes them
            # back into a shared file at their offsets
            path, out_path = extra["path"], extra["out"] + f"{int(extra['cyclic'])}"
            m = hs.DeviceMatrix.load_bspd1(rt, path, cyclic=extra["cyclic"])
            mine = np.zeros_like(a)
            m.download(mine)
            t = torch.from_numpy(mine)
            dist.all_reduce(t)
            dist.barrier()
            m.save_bspd1(out_path)
            dist.barrier()
            out = {"A": t.numpy()}
        elif kind == "refine":
            # mixed-precision solve over the block-cyclic factor: every rank
            # passes full-length vectors and gets the same x
            rhs = o.generate_rhs(n, b, seed=42)
            m = hs.DeviceMatrix(rt, n, b, cyclic=True).upload(a)
            work = hs.DeviceMatrix(rt, n, b, cyclic=True)
            d_rhs = torch.from_numpy(rhs).cuda()
            d_x = torch.zeros_like(d_rhs)
            st = H.solve_spd_refine_device(rt, m, work, d_rhs.data_ptr(), d_x.data_ptr(),
                                           slices=extra.get("slices", 4), max_iters=20)
            out = {"x": d_x.cpu().numpy(), "rel": st.rel_residual, "steps": st.iterations}
        elif kind == "solve":
            # factor + distributed substitutions + distributed residual, then
            # substitutions on an uploaded factor (owned inverses computed)
            rt.set_cholesky_gemm(extra.get("slices", 0))
            rhs = o.generate_rhs(n, b, seed=42)
            m = hs.DeviceMatrix(rt, n, b, cyclic=True).upload(a)
            orig = hs.DeviceMatrix(rt, n, b, cyclic=True).upload(a)
            d_rhs = torch.from_numpy(rhs).cuda()
            d_x = torch.zeros_like(d_rhs)
            rt.ledger(clear=True)
            sp = hs.solve_spd_device(rt, m, d_rhs.data_ptr(), d_x.data_ptr(), a_orig=orig)
            led = [(e.kind, e.step, e.bytes) for e in rt.ledger()]
            _, L, _, _ = o.factorize(n, b, a)
            if extra.get("singular_at") is not None:
                k = extra["singular_at"]
                i = k // b
                L[(i * (i + 1) // 2 + i) * b * b + (k % b) * b + (k % b)] = 0.0
            f = hs.DeviceMatrix(rt, n, b, cyclic=True).upload(L)
            v = d_rhs.clone()
            err = None
            try:
                H.trsv_device(rt, f, v.data_ptr(), False)
                y = v.cpu().numpy()
                H.trsv_device(rt, f, v.data_ptr(), True)
            except hs.SingularBlockError as e:
                err = str(e)
                y = None
            out = {"x": d_x.cpu().numpy(), "res": sp.true_residual, "y": y,
                   "x2": v.cpu().numpy(), "err": err, "ledger": led}
        else:
            rt.set_cholesky_gemm(extra.get("slices", 0))
            if extra.get("break_at"):
                k = extra["break_at"]  # element (k, k) made negative
                N = (n + b - 1) // b
                i = k // b
                a = a.copy()
                a[(i * (i + 1) // 2 + i) * b * b + (k % b) * b + (k % b)] = -5.0
            m = hs.DeviceMatrix(rt, n, b, cyclic=True).upload(a)
            err = None
            try:
                H.potrf_device(rt, m)
            except hs.NotSpdError as e:
                err = (e.block_row, e.pivot_index)
            mine = np.zeros_like(a)
            m.download(mine)  # only this rank's tiles are written
            t = torch.from_numpy(mine)
            dist.all_reduce(t)  # owned tiles are disjoint: the sum is the factor
            out = {"L": t.numpy(), "err": err}
        result_q.put((rank, out))
        rt.close()
    finally:
        dist.destroy_process_group()


def run_ranks(world, job):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, job, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    try:
        for _ in range(world):
            r, out = q.get(timeout=240)
            assert "error" not in out, f"rank {r}:\n{out['error']}"
            res[r] = out
    finally:
        for p in procs:
            p.join(timeout=60)
            if p.is_alive():
                p.kill()
    for p in procs:
        assert p.exitcode == 0
    return res


@pytest.mark.parametrize("world,n,b", [(2, 2048, 128), (3, 1500, 64), (2, 4096, 256),
                                        (4, 4096, 128), (4, 4096, 256), (2, 4096, 512)])
def test_row_sharded_cg_multi_rank(oracle, world, n, b):
    res = run_ranks(world, ("cg", n, b, {}))
    a = oracle.generate_spd(n, b, seed=42)
    ref = oracle.solve_cg(n, b, a, oracle.generate_rhs(n, b, seed=42))
    for r in range(world):  # every rank returns the full x and the same scalars
        out = res[r]
        # the sharded SYMV / rank-ordered dots round differently from the
        # CPU's sequential sums and the CG trace is chaotic:
        # measured up to 3 iterations apart (38 vs 41 at n=4096, b=256),
        # while x agrees to 5e-10
        assert out["conv"] and abs(out["iters"] - ref["iterations"]) <= 4
        assert np.linalg.norm(out["x"][:n] - ref["x"][:n]) <= 1e-6 * np.linalg.norm(ref["x"][:n])
        assert out["res"] <= 2e-6 * np.sqrt(out["u0"])
        assert np.array_equal(out["x"], res[0]["x"])  # identical on every rank


def test_cg_multi_rank_ledger_and_recompute(oracle):
    n, b, iters = 1024, 128, 12
    res = run_ranks(2, ("cg", n, b, {"eps": 1e-300, "max_iters": iters, "recompute": 5}))
    for r in range(2):
        led = res[r]["ledger"]
        assert res[r]["iters"] == iters
        for k in range(1, iters + 1):
            sv = sum(1 for kind, st in led if kind == "subvector" and st == k)
            sc = sum(1 for kind, st in led if kind == "scalar" and st == k)
            # the dot partials ride in the reduce-scatter / all-gather
            assert sc == 0 and sv == 2 + (2 if k % 5 == 0 else 0), (k, sc, sv)


def lower_mask(n, b):
    N = (n + b - 1) // b
    m = np.zeros(N * (N + 1) // 2 * b * b, dtype=bool)
    for i in range(N):
        for j in range(i + 1):
            t = np.tril(np.ones((b, b), dtype=bool)) if i == j else np.ones((b, b), dtype=bool)
            m[(i * (i + 1) // 2 + j) * b * b:(i * (i + 1) // 2 + j + 1) * b * b] = t.ravel()
    return m


@pytest.mark.parametrize("world,n,b,slices", [(2, 2048, 256, 0), (4, 2048, 128, 0),
                                              (4, 4096, 512, 8), (2, 1536, 128, 8)])
def test_block_cyclic_cholesky_multi_rank(oracle, world, n, b, slices):
    res = run_ranks(world, ("chol", n, b, {"slices": slices}))
    a = oracle.generate_spd(n, b, seed=42)
    st, L_ref, _, _ = oracle.factorize(n, b, a)
    mask = lower_mask(n, b)
    for r in range(world):
        assert res[r]["err"] is None
        err = np.abs(res[r]["L"][mask] - L_ref[mask]).max()
        assert err <= 1e-10 * np.abs(a[mask]).max(), (r, err)


def test_block_cyclic_not_spd_agreed_by_all_ranks(oracle):
    n, b = 2048, 256
    res = run_ranks(4, ("chol", n, b, {"break_at": 2 * b + 8}))
    for r in range(4):
        assert res[r]["err"] == (2, 8), res[r]["err"]


@pytest.mark.parametrize("cyclic", [False, True])
def test_multi_rank_bspd1_stream_load_and_save(oracle, tmp_path, cyclic):
    import paper_2605_13209_b200 as hs
    n, b = 1500, 128
    a = oracle.generate_spd(n, b, seed=42)
    path = str(tmp_path / "a.bspd")
    hs.save_matrix(hs.BlockedSPDMatrix(n, b, a.copy()), path)
    out = str(tmp_path / "back")
    res = run_ranks(3, ("io", n, b, {"path": path, "out": out, "cyclic": cyclic}))
    for r in range(3):
        assert res[r]["A"].tobytes() == a.tobytes()
    assert open(out + f"{int(cyclic)}", "rb").read() == open(path, "rb").read()


@pytest.mark.parametrize("world,n,b,slices", [(2, 2048, 256, 0), (4, 2048, 128, 0),
                                              (3, 1500, 128, 8), (4, 4096, 512, 8)])
def test_block_cyclic_solve_multi_rank(oracle, world, n, b, slices):
    """Distributed factor + substitutions + residual, every rank
    returning the same full x; substitutions on an uploaded factor match the
    oracle's forward/back substitution."""
    res = run_ranks(world, ("solve", n, b, {"slices": slices}))
    a = oracle.generate_spd(n, b, seed=42)
    rhs = oracle.generate_rhs(n, b, seed=42)
    ref = oracle.solve_spd(n, b, a, rhs)
    _, y_ref = oracle.forward_substitute(n, b, ref["L"], rhs)
    _, x_ref = oracle.back_substitute(n, b, ref["L"], y_ref)
    nb = np.linalg.norm(rhs)
    N = (n + b - 1) // b
    for r in range(world):
        out = res[r]
        assert np.array_equal(out["x"], res[0]["x"]) and out["res"] == res[0]["res"]
        assert np.linalg.norm(out["x"] - ref["x"]) <= 1e-9 * np.linalg.norm(ref["x"])
        # the reference's own acceptance bound (test_cholesky_solver.cpp:255-269)
        assert out["res"] <= 1e-10 * nb, out["res"] / nb
        assert abs(out["res"] - ref["true_residual"]) <= 1e-10 * nb
        assert np.linalg.norm(out["y"] - y_ref) <= 1e-11 * np.linalg.norm(y_ref)
        assert np.linalg.norm(out["x2"] - x_ref) <= 1e-10 * np.linalg.norm(x_ref)
        # per substitution step: one b-double broadcast; an all-gather of
        # b doubles per rank on every step but the first
        steps = {}
        for kind, st, nbytes in out["ledger"]:
            if kind == "subvector" and st >= 0:
                steps.setdefault(st, []).append(nbytes)
        assert sorted(steps) == list(range(N))
        for st, v in steps.items():
            # forward + backward; the first step of each has no all-gather
            gathers = 2 - (st == 0) - (st == N - 1)
            assert sorted(v) == sorted([b * 8] * 2 + [world * b * 8] * gathers), (st, v)


def test_block_cyclic_substitution_singular_agreed(oracle):
    n, b = 1024, 128
    res = run_ranks(3, ("solve", n, b, {"singular_at": 5 * b + 3}))
    for r in range(3):
        assert res[r]["err"] is not None and res[r]["y"] is None


@pytest.mark.parametrize("world,n,b,slices", [(2, 2048, 256, 4), (4, 2048, 512, 5),
                                              (2, 1536, 128, 0)])
def test_block_cyclic_mixed_precision_refine_multi_rank(oracle, world, n, b, slices):
    """hs_solve_spd_refine over the 2D block-cyclic factor: distributed INT8 /
    DMMA factorization, pipelined substitutions and the all-gathered SYMV in
    each refinement step; every rank ends with the same x, at the FP64
    floor of the residual."""
    res = run_ranks(world, ("refine", n, b, {"slices": slices}))
    a = oracle.generate_spd(n, b, seed=42)
    rhs = oracle.generate_rhs(n, b, seed=42)
    ref = oracle.solve_spd(n, b, a, rhs)
    for r in range(world):
        out = res[r]
        assert out["rel"] <= 1e-10, (r, out["rel"])
        assert np.linalg.norm(out["x"] - ref["x"]) <= 1e-8 * np.linalg.norm(ref["x"])
        assert np.array_equal(out["x"], res[0]["x"]) and out["steps"] == res[0]["steps"]
