"""Python mirror of the reference ``hsolve`` solver API, backed by the B200
C ABI (``libhsolve_cuda.so``).

Names, argument meaning and error behaviour follow the reference headers
(paths relative to /root/reference/proj):

* ``SolverConfig``          solver_config.hpp:12-26 (+ ``gpus``)
* ``KernelParams``          genmat.hpp:14-19
* ``BlockedSPDMatrix``      blocked_matrix.hpp:10-61 (host, packed tiles)
* ``BlockVector``           blocked_matrix.hpp:63-89
* ``Runtime``               executor.hpp:128-221 -> one GPU context
* ``generate_spd`` / ``generate_rhs`` / ``generate_inputs`` /
  ``median_pairwise_distance``                       genmat.hpp:33-45
* ``solve_cg``              cg_solver.hpp:48-49
* ``factorize`` / ``forward_substitute`` / ``back_substitute`` /
  ``solve_spd``             cholesky_solver.hpp:44-58
* ``partition_for_fraction`` / ``cholesky_border``   partition.hpp:20-30
* exceptions                errors.hpp:10-127

Every arithmetic call runs on the GPU through the C ABI; there is no CPU
fallback. Device-resident variants (``DeviceMatrix``, ``solve_cg_device``)
skip host<->device copies for the measured hot path.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from ._lib import CgParams, CgStats, CholStats, RefineStats

# ---------------------------------------------------------------------------
# errors (errors.hpp:10-127; names from transfer_ledger.cpp:28-42)


class HsolveError(RuntimeError):
    kind = "error"


class ConfigError(HsolveError):
    kind = "config_error"


class NotSpdError(HsolveError):
    kind = "not_spd"

    def __init__(self, msg, block_row=-1, pivot_index=-1):
        super().__init__(msg)
        self.block_row = block_row
        self.pivot_index = pivot_index


class SingularBlockError(HsolveError):
    kind = "singular_block"

    def __init__(self, msg, diagonal_index=-1):
        super().__init__(msg)
        self.diagonal_index = diagonal_index


class NumericalError(HsolveError):
    kind = "numerical_error"


class ResidencyError(HsolveError):
    kind = "residency_error"


class FormatError(HsolveError):
    kind = "format_error"


class VersionMismatchError(HsolveError):
    kind = "version_mismatch"

    def __init__(self, msg, expected=-1, actual=-1):
        super().__init__(msg)
        self.expected, self.actual = expected, actual


class TruncatedFileError(HsolveError):
    kind = "truncated_file"

    def __init__(self, msg, expected_bytes=-1, actual_bytes=-1):
        super().__init__(msg)
        self.expected_bytes, self.actual_bytes = expected_bytes, actual_bytes


class IoError(HsolveError):
    kind = "io_error"


class DeviceError(HsolveError):
    kind = "cuda_error"


def _check(status: int) -> None:
    if status == _lib.HS_OK:
        return
    msg, a, b = _lib.last_error()
    if status == _lib.HS_ERR_CONFIG:
        raise ConfigError(msg)
    if status == _lib.HS_ERR_NOT_SPD:
        raise NotSpdError(msg, a, b)
    if status == _lib.HS_ERR_SINGULAR_BLOCK:
        raise SingularBlockError(msg, b)
    if status == _lib.HS_ERR_NUMERICAL:
        raise NumericalError(msg)
    if status == _lib.HS_ERR_RESIDENCY:
        raise ResidencyError(msg)
    if status == _lib.HS_ERR_FORMAT:
        raise FormatError(msg)
    if status == _lib.HS_ERR_VERSION_MISMATCH:
        raise VersionMismatchError(msg, a, b)
    if status == _lib.HS_ERR_TRUNCATED_FILE:
        raise TruncatedFileError(msg, a, b)
    if status == _lib.HS_ERR_IO:
        raise IoError(msg)
    raise DeviceError(f"status {status}: {msg}")


# ---------------------------------------------------------------------------
# configuration


@dataclass
class SolverConfig:
    eps: float = 1e-6
    max_iters: int = 500
    recompute_interval: int = 50
    fraction: float = 0.0
    block_size: int = 32
    workers_a: int = 2
    workers_b: int = 2
    slowdown_a: float = 1.0
    slowdown_b: float = 1.0
    seed: int = 42
    record_trace: bool = False
    gpus: int = 1  # B200 build: number of GPUs the work is partitioned over
    comm: int = 0  # multi-GPU collectives: 0 auto, 1 NCCL, 2 in-process copies

    def validate(self) -> None:  # solver_config.cpp:9-26
        if not (self.eps > 0.0):
            raise ConfigError(f"eps must be positive, got {self.eps}")
        if not (0.0 <= self.fraction <= 1.0):
            raise ConfigError(f"fraction must be in [0, 1], got {self.fraction}")
        if self.block_size == 0:
            raise ConfigError("block size must be positive")
        if self.workers_a == 0 or self.workers_b == 0:
            raise ConfigError("both executors need at least one worker")
        if not (self.slowdown_a >= 1.0) or not (self.slowdown_b >= 1.0):
            raise ConfigError("slowdown factors must be >= 1.0")
        if self.gpus < 1:
            raise ConfigError("gpus must be >= 1")
        if self.comm not in (0, 1, 2):
            raise ConfigError("comm must be 0 (auto), 1 (NCCL) or 2 (in-process)")


@dataclass
class KernelParams:
    sigma_f2: float = 1.0
    length_scale: float = 0.0  # <= 0: median pairwise distance rule
    sigma_n2: float = 1e-2
    dim: int = 2


# ---------------------------------------------------------------------------
# host storage (same layout as the reference)


def block_rows(n: int, b: int) -> int:
    return (n + b - 1) // b


def block_index(i: int, j: int, rows: int) -> int:  # blocked_matrix.cpp:8-15
    if i >= rows or j > i:
        raise IndexError(f"block_index({i}, {j}) out of range for {rows} block rows")
    return i * (i + 1) // 2 + j


class BlockedSPDMatrix:
    """Packed lower-triangular b x b tiles, row-major inside a tile, identity
    padding of rows/cols >= n (blocked_matrix.hpp:10-61)."""

    def __init__(self, n: int, b: int, values: np.ndarray | None = None):
        if n == 0 or b == 0:
            raise ConfigError("matrix size and block size must be positive")
        self.n, self.b = int(n), int(b)
        self.rows = block_rows(n, b)
        cnt = self.block_count * b * b
        if values is None:
            self.values = np.zeros(cnt)
            self.apply_identity_padding()
        else:
            v = np.ascontiguousarray(values, dtype=np.float64)
            if v.size != cnt:
                raise ConfigError(f"expected {cnt} packed values, got {v.size}")
            self.values = v

    @property
    def block_count(self) -> int:
        return self.rows * (self.rows + 1) // 2

    @property
    def padded_n(self) -> int:
        return self.rows * self.b

    def block(self, i: int, j: int) -> np.ndarray:
        k = block_index(i, j, self.rows)
        b = self.b
        return self.values[k * b * b:(k + 1) * b * b].reshape(b, b)

    def element(self, p: int, q: int) -> float:
        if p >= self.n or q >= self.n:
            raise IndexError(f"element({p}, {q}) out of range for n = {self.n}")
        if p < q:
            p, q = q, p
        return float(self.block(p // self.b, q // self.b)[p % self.b, q % self.b])

    def set(self, p: int, q: int, value: float) -> None:
        if p >= self.n or q >= self.n:
            raise IndexError(f"set({p}, {q}) out of range for n = {self.n}")
        if p < q:
            p, q = q, p
        self.block(p // self.b, q // self.b)[p % self.b, q % self.b] = value

    def apply_identity_padding(self) -> None:  # blocked_matrix.cpp:57-74
        pad = self.padded_n - self.n
        if pad == 0:
            return
        last, b = self.rows - 1, self.b
        for j in range(self.rows):
            d = self.block(last, j)
            for r in range(b):
                p = last * b + r
                if p < self.n:
                    continue
                d[r, :] = 0.0
                q0 = j * b
                if q0 <= p < q0 + b:
                    d[r, p - q0] = 1.0

    @staticmethod
    def identity(n: int, b: int) -> "BlockedSPDMatrix":
        m = BlockedSPDMatrix(n, b)
        for i in range(m.rows):
            np.fill_diagonal(m.block(i, i), 1.0)
        return m

    def copy(self) -> "BlockedSPDMatrix":
        return BlockedSPDMatrix(self.n, self.b, self.values.copy())

    def to_dense(self) -> np.ndarray:
        """Logical n x n symmetric image (reads the canonical lower tiles)."""
        n, b, N = self.n, self.b, self.rows
        pn = N * b
        d = np.zeros((pn, pn))
        for i in range(N):
            for j in range(i + 1):
                d[i * b:(i + 1) * b, j * b:(j + 1) * b] = self.block(i, j)
        lo = np.tril(d)
        return (lo + np.tril(lo, -1).T)[:n, :n]


class BlockVector:
    """N*b doubles with a zero padded tail (blocked_matrix.hpp:63-89)."""

    def __init__(self, n: int, b: int, values: np.ndarray | None = None):
        if n == 0 or b == 0:
            raise ConfigError("vector size and block size must be positive")
        self.n, self.b = int(n), int(b)
        self.rows = block_rows(n, b)
        if values is None:
            self.values = np.zeros(self.rows * b)
        else:
            v = np.ascontiguousarray(values, dtype=np.float64)
            if v.size == n and n != self.rows * b:
                full = np.zeros(self.rows * b)
                full[:n] = v
                v = full
            if v.size != self.rows * b:
                raise ConfigError("vector length does not match the blocking")
            self.values = v

    @property
    def padded_n(self) -> int:
        return self.rows * self.b

    def __getitem__(self, i):
        return self.values[i]

    def __setitem__(self, i, v):
        self.values[i] = v

    def logical(self) -> np.ndarray:
        return self.values[: self.n]


# ---------------------------------------------------------------------------
# runtime = GPU context (executor.hpp:128-221)


class Runtime:
    """One GPU context (device + stream, optional NCCL communicator).

    ``Runtime(cfg)`` mirrors the reference constructor; ``workers_*`` and
    ``slowdown_*`` are accepted for compatibility and have no effect.
    """

    def __init__(self, cfg: SolverConfig | None = None, device: int = 0,
                 stream: int | None = None, _handle=None):
        if cfg is not None:
            cfg.validate()
        self._L = _lib.lib()
        self.group = None
        gpus = cfg.gpus if cfg is not None else 1
        if _handle is None and gpus > 1:
            # one process, G GPUs (hs_group): rank r on device (device + r) % count
            cnt = C.c_int(0)
            _check(self._L.hs_device_count(C.byref(cnt)))
            devs = (C.c_int * gpus)(*[(device + r) % max(cnt.value, 1) for r in range(gpus)])
            g = C.c_void_p()
            _check(self._L.hs_group_create(gpus, devs, cfg.comm, C.byref(g)))
            self.group = g
            _handle = C.c_void_p(self._L.hs_group_ctx(g, 0))
        if _handle is not None:
            self.ctx = _handle
        else:
            h = C.c_void_p()
            _check(self._L.hs_ctx_create(device, C.c_void_p(stream or 0), C.byref(h)))
            self.ctx = h
        self.device = device
        import weakref
        self._matrices = weakref.WeakSet()  # freed before the context closes

    @classmethod
    def distributed(cls, device: int, rank: int, world: int, nccl_id: bytes,
                    stream: int | None = None) -> "Runtime":
        L = _lib.lib()
        h = C.c_void_p()
        buf = C.create_string_buffer(bytes(nccl_id), 128)
        _check(L.hs_ctx_create_nccl(device, C.c_void_p(stream or 0), rank, world, buf,
                                    C.byref(h)))
        return cls(device=device, _handle=h)

    @classmethod
    def custom_comm(cls, device: int, rank: int, world: int, transport,
                    stream: int | None = None) -> "Runtime":
        """Multi-rank context whose collectives go through ``transport``, an
        object with ``allgather(send_ptr, recv_ptr, count)``,
        ``reduce_scatter(send_ptr, recv_ptr, count)``,
        ``broadcast(send_ptr, recv_ptr, count, root)`` and
        ``allreduce_max_i64(ptr, count)`` on device pointers (see
        hs_ctx_create_custom_comm; a test transport, not a fast one)."""
        L = _lib.lib()

        def wrap(fn):
            def cb(*args):
                try:
                    fn(*args[1:])
                    return 0
                except Exception:  # the C side turns non-zero into an error
                    import traceback
                    traceback.print_exc()
                    return 1
            return cb

        ops = _lib.CommOps(_lib.ALLGATHER_FN(wrap(transport.allgather)),
                           _lib.REDUCE_SCATTER_FN(wrap(transport.reduce_scatter)),
                           _lib.BROADCAST_FN(wrap(transport.broadcast)),
                           _lib.ALLREDUCE_MAX_FN(wrap(transport.allreduce_max_i64)), None)
        h = C.c_void_p()
        _check(L.hs_ctx_create_custom_comm(device, C.c_void_p(stream or 0), rank, world,
                                           C.byref(ops), C.byref(h)))
        rt = cls(device=device, _handle=h)
        rt._ops = ops  # keep the callbacks alive with the context
        return rt

    @staticmethod
    def nccl_unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        _check(_lib.lib().hs_nccl_unique_id(buf))
        return buf.raw

    @property
    def rank(self) -> int:
        return self._L.hs_ctx_rank(self.ctx)

    @property
    def world(self) -> int:
        return self._L.hs_ctx_world(self.ctx)

    @property
    def stream(self) -> int:
        return self._L.hs_ctx_stream(self.ctx) or 0

    def kernel_launches(self) -> int:
        return int(self._L.hs_ctx_kernel_launches(self.ctx))

    def set_cholesky_gemm(self, slices: int) -> None:
        """Cholesky trailing-update engine: 0 = FP64 DMMA (default), 1..8 =
        FP64 emulated on the INT8 tensor cores with that many slices."""
        if self.group:
            _check(self._L.hs_group_set_cholesky_gemm(self.group, int(slices)))
        else:
            _check(self._L.hs_ctx_set_cholesky_gemm(self.ctx, int(slices)))

    def trim(self) -> None:
        """Release cached device matrices / workspaces (hs_ctx_trim)."""
        _check(self._L.hs_ctx_trim(self.ctx))

    def close(self) -> None:
        if getattr(self, "ctx", None):
            for m in list(getattr(self, "_matrices", ())):
                m.free()
            if getattr(self, "group", None):
                self._L.hs_group_destroy(self.group)
                self.group = None
            else:
                self._L.hs_ctx_destroy(self.ctx)
            self.ctx = None

    @property
    def gpus(self) -> int:
        return self._L.hs_group_world(self.group) if self.group else 1

    @property
    def transport(self) -> str:
        """Collectives of a multi-GPU Runtime: "nccl", "in-process" or "none"."""
        if not self.group:
            return "none"
        return {0: "none", 1: "nccl", 2: "in-process"}[self._L.hs_group_transport(self.group)]

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # profiling hooks used by bench.py
    def prof_enable(self, every: int = 1) -> None:
        """Bracket every `every`-th SYMV launch with CUDA events (0: off)."""
        self._L.hs_prof_enable(self.ctx, int(every))

    def prof_symv(self) -> tuple[int, float]:
        n, ms = C.c_uint64(0), C.c_double(0.0)
        self._L.hs_prof_symv(self.ctx, C.byref(n), C.byref(ms))
        return int(n.value), float(ms.value)

    def prof_reset(self) -> None:
        self._L.hs_prof_reset(self.ctx)

    # communication ledger (transfer_ledger.hpp): one entry per NCCL collective
    def ledger(self, clear: bool = False) -> list[TransferEntry]:
        k = int(self._L.hs_ctx_ledger_size(self.ctx))
        buf = (_lib.LedgerEntry * max(k, 1))()
        k = int(self._L.hs_ctx_ledger_read(self.ctx, buf, k))
        out = [TransferEntry(TRANSFER_KINDS[e.kind], DIRECTIONS[e.direction], int(e.bytes),
                             int(e.step)) for e in buf[:k]]
        if clear:
            self._L.hs_ctx_ledger_clear(self.ctx)
        return out


TRANSFER_KINDS = ("scalar", "subvector", "block", "block_row", "initial_matrix", "result")
DIRECTIONS = ("a_to_b", "b_to_a", "bidirectional")


@dataclass
class TransferEntry:  # transfer_ledger.hpp:28-33
    kind: str
    direction: str
    bytes: int
    step: int


_DEFAULT_RT: Runtime | None = None


def default_runtime() -> Runtime:
    global _DEFAULT_RT
    if _DEFAULT_RT is None:
        _DEFAULT_RT = Runtime()
    return _DEFAULT_RT


# ---------------------------------------------------------------------------
# device-resident matrix


class DeviceMatrix:
    """Packed tiles resident in HBM: this rank's block rows (CG layout) or,
    with ``cyclic=True``, its tiles of the 2D block-cyclic distribution used
    by the multi-GPU Cholesky."""

    def __init__(self, rt: Runtime, n: int, b: int, cyclic: bool = False):
        self.rt, self.n, self.b = rt, int(n), int(b)
        self.rows = block_rows(n, b)
        h = C.c_void_p()
        create = rt._L.hs_matrix_create_cyclic if cyclic else rt._L.hs_matrix_create
        _check(create(rt.ctx, n, b, C.byref(h)))
        self.h = h
        rt._matrices.add(self)
        lo, hi = C.c_size_t(), C.c_size_t()
        _check(rt._L.hs_matrix_info(h, None, None, C.byref(lo), C.byref(hi)))
        self.row_lo, self.row_hi = lo.value, hi.value

    @property
    def packed_len(self) -> int:
        return self.rows * (self.rows + 1) // 2 * self.b * self.b

    def upload(self, host: BlockedSPDMatrix | np.ndarray) -> "DeviceMatrix":
        v = host.values if isinstance(host, BlockedSPDMatrix) else np.ascontiguousarray(host)
        assert v.dtype == np.float64 and v.size == self.packed_len
        _check(self.rt._L.hs_matrix_upload(self.h, v.ctypes.data))
        return self

    def download(self, out: np.ndarray | None = None) -> np.ndarray:
        if out is None:
            out = np.zeros(self.packed_len)
        _check(self.rt._L.hs_matrix_download(self.h, out.ctypes.data))
        return out

    def to_host(self) -> BlockedSPDMatrix:
        return BlockedSPDMatrix(self.n, self.b, self.download())

    def copy_from(self, other: "DeviceMatrix") -> "DeviceMatrix":
        _check(self.rt._L.hs_matrix_copy(self.h, other.h))
        return self

    def data_ptr(self) -> int:
        return self.rt._L.hs_matrix_device_data(self.h) or 0

    @classmethod
    def load_bspd1(cls, rt: Runtime, path: str, cyclic: bool = False) -> "DeviceMatrix":
        """Stream a BSPD1 file into HBM tiles (no host copy of the matrix)."""
        h = C.c_void_p()
        _check(rt._L.hs_matrix_load_bspd1(rt.ctx, os.fsencode(path), int(cyclic),
                                          C.byref(h)))
        self = cls.__new__(cls)
        self.rt, self.h = rt, h
        n, b, lo, hi = C.c_size_t(), C.c_size_t(), C.c_size_t(), C.c_size_t()
        _check(rt._L.hs_matrix_info(h, C.byref(n), C.byref(b), C.byref(lo), C.byref(hi)))
        self.n, self.b = n.value, b.value
        self.rows = block_rows(self.n, self.b)
        self.row_lo, self.row_hi = lo.value, hi.value
        rt._matrices.add(self)
        return self

    def save_bspd1(self, path: str) -> None:
        _check(self.rt._L.hs_matrix_save_bspd1(self.h, os.fsencode(path)))

    def assemble_se(self, points: np.ndarray, dim: int, sigma_f2: float, inv2l2: float,
                    sigma_n2: float) -> None:
        p = np.ascontiguousarray(points, dtype=np.float64)
        _check(self.rt._L.hs_assemble_se(self.h, p.ctypes.data, dim, sigma_f2, inv2l2,
                                         sigma_n2))

    def free(self) -> None:
        if getattr(self, "h", None):
            if self.rt.ctx is not None:  # the context owns the device memory
                self.rt._L.hs_matrix_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


# ---------------------------------------------------------------------------
# generators (genmat.hpp)


def generate_inputs(n: int, dim: int, seed: int) -> np.ndarray:
    out = np.zeros(n * dim)
    _check(_lib.lib().hs_generate_inputs(n, dim, seed, out.ctypes.data))
    return out


def median_pairwise_distance(points: np.ndarray, n: int, dim: int) -> float:
    p = np.ascontiguousarray(points, dtype=np.float64)
    return float(_lib.lib().hs_median_pairwise_distance(p.ctypes.data, n, dim))


def generate_rhs(n: int, b: int, seed: int) -> BlockVector:
    v = BlockVector(n, b)
    _check(_lib.lib().hs_generate_rhs(n, b, seed, v.values.ctypes.data))
    return v


def generate_spd_device(rt: Runtime, n: int, b: int, params: KernelParams | None = None,
                        seed: int = 42, cyclic: bool = False) -> DeviceMatrix:
    """GP squared-exponential matrix assembled on the GPU (never on the host);
    each rank assembles only the tiles it owns."""
    p = params or KernelParams()
    m = DeviceMatrix(rt, n, b, cyclic=cyclic)
    _check(rt._L.hs_generate_spd(m.h, p.sigma_f2, p.length_scale, p.sigma_n2, p.dim,
                                 seed))
    return m


def generate_spd(n: int, b: int, params: KernelParams | None = None, seed: int = 42,
                 rt: Runtime | None = None) -> BlockedSPDMatrix:
    """genmat.hpp:41-42: tiles generated on the GPU, returned as host storage."""
    p = params or KernelParams()
    if not (p.sigma_f2 > 0.0) or not (p.sigma_n2 > 0.0):
        raise ConfigError("kernel variances must be positive")
    m = generate_spd_device(rt or default_runtime(), n, b, p, seed)
    try:
        return m.to_host()
    finally:
        m.free()


# ---------------------------------------------------------------------------
# work split (partition.hpp)


@dataclass
class Partition:
    split_row: int = 0
    fraction: float = 0.0


def partition_for_fraction(fraction: float, rows: int) -> Partition:
    out = C.c_size_t()
    _check(_lib.lib().hs_partition_for_fraction(fraction, rows, C.byref(out)))
    return Partition(out.value, fraction)


def cholesky_border(fraction: float, column: int, rows: int) -> int:
    out = C.c_size_t()
    _check(_lib.lib().hs_cholesky_border(fraction, column, rows, C.byref(out)))
    return out.value


def partition_rows(rows: int, world: int) -> list[int]:
    out = np.zeros(world + 1, dtype=np.uint64)
    _check(_lib.lib().hs_partition_rows(rows, world, out.ctypes.data))
    return [int(v) for v in out]


# ---------------------------------------------------------------------------
# CG (cg_solver.hpp)


@dataclass
class CgIteration:
    u: float
    alpha: float
    beta: float


@dataclass
class CgStatsPy:
    iterations: int = 0
    recomputations: int = 0
    converged: bool = False
    u0: float = 0.0
    true_residual: float = 0.0
    wall_ms: float = 0.0
    compute_ms: float = 0.0
    transfer_ms: float = 0.0
    partition: Partition = field(default_factory=Partition)
    trace: list = field(default_factory=list)


@dataclass
class CgResult:
    x: BlockVector
    stats: CgStatsPy


def _cg_params(cfg: SolverConfig) -> CgParams:
    return CgParams(cfg.eps, cfg.max_iters, cfg.recompute_interval,
                    1 if cfg.record_trace else 0)


def _cg_stats(st: CgStats, tr: np.ndarray | None, cfg: SolverConfig, rows: int,
              gpus: int = 1) -> CgStatsPy:
    out = CgStatsPy(int(st.iterations), int(st.recomputations), bool(st.converged),
                    st.u0, st.true_residual, st.wall_ms, st.compute_ms, st.transfer_ms)
    # the split that ran: rank 0's block rows of a 2-GPU Runtime (clamped to
    # [1, N-1]); none on one GPU
    split = 0
    if gpus == 2 and 0.0 < cfg.fraction < 1.0 and rows >= 2:
        split = min(max(partition_for_fraction(cfg.fraction, rows).split_row, 1), rows - 1)
    out.partition = Partition(split, cfg.fraction)
    if tr is not None:
        k = out.iterations
        out.trace = [CgIteration(*tr[3 * i:3 * i + 3]) for i in range(k)]
    return out


def _shape_check(a, rhs) -> None:
    if rhs.n != a.n or rhs.b != a.b:
        raise ConfigError("matrix and right-hand side shapes do not match")


def solve_cg(a: BlockedSPDMatrix, rhs: BlockVector, cfg: SolverConfig,
             rt: Runtime | None = None) -> CgResult:
    """cg_solver.hpp:48-49 with HOST buffers (H2D / D2H inside the call)."""
    cfg.validate()
    _shape_check(a, rhs)
    if cfg.block_size != a.b:
        raise ConfigError("config block size does not match the matrix")
    rt = rt or default_runtime()
    x = BlockVector(a.n, a.b)
    st = CgStats()
    tr = np.zeros(3 * max(cfg.max_iters, 1)) if cfg.record_trace else None
    p = _cg_params(cfg)
    if rt.group:
        _check(rt._L.hs_group_set_row_fraction(rt.group, cfg.fraction))
        _check(rt._L.hs_group_solve_cg_host(rt.group, a.n, a.b, a.values.ctypes.data,
                                            rhs.values.ctypes.data, C.byref(p),
                                            x.values.ctypes.data, C.byref(st),
                                            tr.ctypes.data if tr is not None else None))
    else:
        _check(rt._L.hs_solve_cg_host(rt.ctx, a.n, a.b, a.values.ctypes.data,
                                      rhs.values.ctypes.data, C.byref(p), x.values.ctypes.data,
                                      C.byref(st), tr.ctypes.data if tr is not None else None))
    return CgResult(x, _cg_stats(st, tr, cfg, a.rows, rt.gpus))


def solve_cg_device(rt: Runtime, a: DeviceMatrix, d_rhs: int, d_x: int,
                    cfg: SolverConfig) -> CgStatsPy:
    """Device-resident CG: d_rhs / d_x are device pointers of N*b doubles."""
    cfg.validate()
    st = CgStats()
    tr = np.zeros(3 * max(cfg.max_iters, 1)) if cfg.record_trace else None
    p = _cg_params(cfg)
    _check(rt._L.hs_cg_solve(rt.ctx, a.h, C.c_void_p(d_rhs), C.byref(p), C.c_void_p(d_x),
                             C.byref(st), tr.ctypes.data if tr is not None else None))
    return _cg_stats(st, tr, cfg, a.rows)


def symv_device(rt: Runtime, a: DeviceMatrix, d_x: int, d_y: int) -> None:
    _check(rt._L.hs_symv(rt.ctx, a.h, C.c_void_p(d_x), C.c_void_p(d_y)))


def true_residual_device(rt: Runtime, a: DeviceMatrix, d_x: int, d_rhs: int) -> float:
    out = C.c_double()
    _check(rt._L.hs_true_residual(rt.ctx, a.h, C.c_void_p(d_x), C.c_void_p(d_rhs),
                                  C.byref(out)))
    return out.value


# ---------------------------------------------------------------------------
# Cholesky (cholesky_solver.hpp)


@dataclass
class FactorizeStats:
    factor_ms: float = 0.0
    compute_ms: float = 0.0
    transfer_ms: float = 0.0


@dataclass
class SpdSolveStats:
    factor_ms: float = 0.0
    solve_ms: float = 0.0
    wall_ms: float = 0.0
    compute_ms: float = 0.0
    transfer_ms: float = 0.0
    true_residual: float = 0.0


@dataclass
class SpdSolveResult:
    x: BlockVector
    stats: SpdSolveStats


def factorize(a: BlockedSPDMatrix, cfg: SolverConfig, rt: Runtime | None = None
              ) -> FactorizeStats:
    """In place: the lower tiles of ``a`` hold L afterwards."""
    cfg.validate()
    rt = rt or default_runtime()
    st = CholStats()
    if rt.group:
        _check(rt._L.hs_group_factorize_host(rt.group, a.n, a.b, a.values.ctypes.data,
                                             C.byref(st)))
    else:
        _check(rt._L.hs_factorize_host(rt.ctx, a.n, a.b, a.values.ctypes.data, C.byref(st)))
    return FactorizeStats(st.factor_ms, st.compute_ms, st.transfer_ms)


def forward_substitute(l: BlockedSPDMatrix, rhs: BlockVector, rt: Runtime | None = None
                       ) -> BlockVector:
    _shape_check(l, rhs)
    rt = rt or default_runtime()
    y = BlockVector(l.n, l.b)
    _check(rt._L.hs_forward_substitute_host(rt.ctx, l.n, l.b, l.values.ctypes.data,
                                            rhs.values.ctypes.data, y.values.ctypes.data))
    return y


def back_substitute(l: BlockedSPDMatrix, y: BlockVector, rt: Runtime | None = None
                    ) -> BlockVector:
    _shape_check(l, y)
    rt = rt or default_runtime()
    x = BlockVector(l.n, l.b)
    _check(rt._L.hs_back_substitute_host(rt.ctx, l.n, l.b, l.values.ctypes.data,
                                         y.values.ctypes.data, x.values.ctypes.data))
    return x


def solve_spd(a: BlockedSPDMatrix, rhs: BlockVector, cfg: SolverConfig,
              rt: Runtime | None = None) -> SpdSolveResult:
    """factorize + substitutions; destroys ``a`` (holds L)."""
    cfg.validate()
    _shape_check(a, rhs)
    rt = rt or default_runtime()
    x = BlockVector(a.n, a.b)
    st = CholStats()
    f = (lambda *a_: rt._L.hs_group_solve_spd_host(rt.group, *a_)) if rt.group else (
        lambda *a_: rt._L.hs_solve_spd_host(rt.ctx, *a_))
    _check(f(a.n, a.b, a.values.ctypes.data, rhs.values.ctypes.data, x.values.ctypes.data,
             C.byref(st)))
    return SpdSolveResult(x, SpdSolveStats(st.factor_ms, st.solve_ms, st.wall_ms,
                                           st.compute_ms, st.transfer_ms, st.true_residual))


def potrf_device(rt: Runtime, a: DeviceMatrix) -> FactorizeStats:
    st = CholStats()
    _check(rt._L.hs_potrf(rt.ctx, a.h, C.byref(st)))
    return FactorizeStats(st.factor_ms, st.compute_ms, 0.0)


def trsv_device(rt: Runtime, l: DeviceMatrix, d_v: int, upper: bool) -> None:
    f = rt._L.hs_trsv_upper if upper else rt._L.hs_trsv_lower
    _check(f(rt.ctx, l.h, C.c_void_p(d_v)))


def solve_spd_device(rt: Runtime, a: DeviceMatrix, d_rhs: int, d_x: int,
                     a_orig: DeviceMatrix | None = None) -> SpdSolveStats:
    st = CholStats()
    _check(rt._L.hs_solve_spd(rt.ctx, a.h, C.c_void_p(d_rhs), C.c_void_p(d_x),
                              a_orig.h if a_orig is not None else None, C.byref(st)))
    return SpdSolveStats(st.factor_ms, st.solve_ms, st.wall_ms, st.compute_ms, 0.0,
                         st.true_residual)


@dataclass
class RefineSolveStats:
    factor_ms: float = 0.0
    solve_ms: float = 0.0
    wall_ms: float = 0.0
    rel_residual: float = 0.0
    iterations: int = 0
    slices: int = 0


def solve_spd_refine_device(rt: Runtime, a: DeviceMatrix, work: DeviceMatrix, d_rhs: int,
                            d_x: int, slices: int = 5, max_iters: int = 10,
                            tol: float = 0.0) -> RefineSolveStats:
    """Mixed-precision SPD solve (hs_solve_spd_refine): factor a copy of A into
    `work` with `slices` Ozaki slices on the INT8 tensor cores (0 = FP64 DMMA),
    then FP64 iterative refinement against the unmodified A until
    ||rhs - A x|| <= tol ||rhs||, max_iters steps, or a step that does not
    halve the residual (tol = 0: refine to the FP64 floor). Beyond the
    reference API (the paper's future-work direction)."""
    st = RefineStats()
    _check(rt._L.hs_solve_spd_refine(rt.ctx, a.h, work.h, C.c_void_p(d_rhs), C.c_void_p(d_x),
                                     int(slices), int(max_iters), float(tol), C.byref(st)))
    return RefineSolveStats(st.factor_ms, st.solve_ms, st.wall_ms, st.rel_residual,
                            st.iterations, st.slices)


# single-tile kernels (block_kernels.hpp:17-31), batched on the device
def potf_tiles_device(rt: Runtime, d_tiles: int, b: int, count: int) -> None:
    piv = C.c_int64(-1)
    _check(rt._L.hs_potf_tiles(rt.ctx, C.c_void_p(d_tiles), b, count, C.byref(piv)))


def gemm_update_tiles_device(rt: Runtime, d_c: int, d_p: int, d_q: int, b: int, count: int,
                             lower_only: bool = False) -> None:
    _check(rt._L.hs_gemm_update_tiles(rt.ctx, C.c_void_p(d_c), C.c_void_p(d_p),
                                      C.c_void_p(d_q), b, count, 1 if lower_only else 0))


# ---------------------------------------------------------------------------
# BSPD1 files (matrix_io.hpp:9-19), host side; DeviceMatrix.load_bspd1 /
# save_bspd1 stream the same format straight to / from HBM.


def save_matrix(m: BlockedSPDMatrix, path: str) -> None:
    v = np.ascontiguousarray(m.values, dtype=np.float64)
    _check(_lib.lib().hs_bspd1_write(os.fsencode(path), m.n, m.b, v.ctypes.data))


def load_matrix(path: str) -> BlockedSPDMatrix:
    L = _lib.lib()
    n, b = C.c_size_t(), C.c_size_t()
    _check(L.hs_bspd1_probe(os.fsencode(path), C.byref(n), C.byref(b)))
    m = BlockedSPDMatrix(n.value, b.value)
    _check(L.hs_bspd1_read(os.fsencode(path), m.values.ctypes.data, m.values.size))
    return m


def save_vector(v: BlockVector, path: str) -> None:
    _check(_lib.lib().hs_vector_write(os.fsencode(path), v.n, v.values.ctypes.data))


def load_vector(path: str, block_size: int) -> BlockVector:
    L = _lib.lib()
    n = C.c_size_t()
    _check(L.hs_vector_probe(os.fsencode(path), C.byref(n)))
    v = BlockVector(n.value, block_size)
    _check(L.hs_vector_read(os.fsencode(path), v.values.ctypes.data, n.value))
    return v
