/*
 * hs_cuda.h — C ABI of libhsolve_cuda.so, the B200-native (sm_100a) SPD-solve
 * path: GP squared-exponential assembly, blocked CG, tiled right-looking
 * Cholesky with triangular solves.
 *
 * This is the drop-in boundary for the reference `hsolve` solver API (paths
 * relative to /root/reference/proj). The reference has no FFI; its boundary
 * is the C++ header API called by bench.cpp:108-126 and the tests. Every
 * entry point below names the reference interface it replaces. The C++ shim
 * in include/hsolve/ (libhsolve_b200.so) re-exposes the reference signatures
 * verbatim on top of this ABI; Python reaches it through ctypes
 * (paper_2605_13209_b200/_lib.py).
 *
 * Conventions
 *  - Plain pointers and sizes only; no exceptions cross the ABI.
 *  - Every call returns an hs_status: 0 = ok, else 1 + hsolve::ErrorKind
 *    (errors.hpp:10-21) or HS_ERR_CUDA for device/runtime failures.
 *    hs_last_error() gives the message, hs_last_error_payload() the payload
 *    (not_spd: block row + pivot, errors.hpp:45-63; numerical: iteration).
 *  - "host" pointers are ordinary (pageable or pinned) host memory; "d_"
 *    pointers are device memory on the context's GPU.
 *  - Layouts are the reference's: packed lower-triangular b x b tiles,
 *    tile (i, j) at (i(i+1)/2 + j) * b * b, row-major inside a tile
 *    (blocked_matrix.hpp:10-61); vectors are N*b doubles with a zero tail
 *    (blocked_matrix.hpp:63-89). N = ceil(n / b).
 *  - Calls are blocking with respect to the host (the reference's barrier()
 *    semantics, executor.hpp:160-162) unless documented otherwise; work is
 *    ordered on the context's stream.
 */
#ifndef HS_CUDA_H
#define HS_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef int hs_status;

enum {
  HS_OK = 0,
  HS_ERR_CONFIG = 1,         /* ErrorKind::config         */
  HS_ERR_NOT_SPD = 2,        /* ErrorKind::not_spd        */
  HS_ERR_SINGULAR_BLOCK = 3, /* ErrorKind::singular_block */
  HS_ERR_NUMERICAL = 4,      /* ErrorKind::numerical      */
  HS_ERR_NOT_CONVERGED = 5,  /* status only; never returned by a solve */
  HS_ERR_RESIDENCY = 6,      /* ErrorKind::residency (never produced)  */
  HS_ERR_FORMAT = 7,         /* ErrorKind::format                      */
  HS_ERR_VERSION_MISMATCH = 8, /* ErrorKind::version_mismatch: payload (expected, actual) */
  HS_ERR_TRUNCATED_FILE = 9, /* ErrorKind::truncated_file: payload (expected, actual bytes) */
  HS_ERR_IO = 10,            /* ErrorKind::io                          */
  HS_ERR_CUDA = 100          /* device / runtime failure (no reference kind) */
};

typedef struct hs_ctx hs_ctx;       /* one GPU + stream (+ NCCL comm) */
typedef struct hs_matrix hs_matrix; /* device-resident packed tiles   */

/* ---- errors ------------------------------------------------------------ */
const char* hs_last_error(void);
void hs_last_error_payload(int64_t* a, int64_t* b);
const char* hs_error_kind_name(hs_status s); /* transfer_ledger.cpp:28-42 */

/* ---- context (replaces hsolve::Runtime, executor.hpp:128-221) ---------- */
hs_status hs_device_count(int* count); /* visible CUDA devices */
/* Device buffers on the context's GPU for FFI callers without a CUDA
 * runtime of their own; hs_memcpy copies any direction (unified addressing)
 * and returns when the copy is done. */
hs_status hs_device_alloc(hs_ctx* ctx, size_t bytes, void** out);
void hs_device_free(hs_ctx* ctx, void* p);
hs_status hs_memcpy(hs_ctx* ctx, void* dst, const void* src, size_t bytes);
/* stream: a cudaStream_t to order work on (NULL = the library creates one). */
hs_status hs_ctx_create(int device, void* stream, hs_ctx** out);
/* Multi-GPU: one process per GPU; nccl_id = 128 bytes from
 * hs_nccl_unique_id() on rank 0, distributed by the caller. */
hs_status hs_nccl_unique_id(void* id128);
hs_status hs_ctx_create_nccl(int device, void* stream, int rank, int world,
                             const void* id128, hs_ctx** out);
/* Multi-rank context over caller-provided collectives instead of NCCL: the
 * SAME distributed CG / Cholesky code paths, with every collective handed to
 * a host callback (device pointers on the context's GPU; the library
 * synchronizes the issuing stream first, and the callback must complete the
 * operation -- e.g. D2H, a gloo collective, H2D -- before returning, status 0
 * on success). Lets several processes share one GPU as separate ranks (NCCL
 * refuses duplicate GPUs), which is how the world > 1 paths are tested on a
 * single-GPU box; it is not a performance transport. */
typedef struct {
  int (*allgather)(void* user, const double* send, double* recv, size_t count);
  int (*reduce_scatter)(void* user, const double* send, double* recv, size_t count);
  int (*broadcast)(void* user, const double* send, double* recv, size_t count, int root);
  int (*allreduce_max_i64)(void* user, int64_t* buf, size_t count);
  void* user;
} hs_comm_ops;
hs_status hs_ctx_create_custom_comm(int device, void* stream, int rank, int world,
                                    const hs_comm_ops* ops, hs_ctx** out);
void hs_ctx_destroy(hs_ctx* ctx);

/* ---- single-process multi-GPU group (hsolve::Runtime with gpus > 1) ----
 * The reference's Runtime drives its two executors from one orchestrator
 * (executor.hpp:122-132); a group drives G ranks from one process: one
 * hs_ctx per rank (rank r on devices[r], or device r % count when NULL) and
 * one host thread per rank while a solve runs. transport: 0 = auto (NCCL via
 * ncclCommInitAll when every rank has its own device, else in-process),
 * 1 = NCCL, 2 = in-process (collectives are event-ordered device copies
 * between the ranks' buffers: asynchronous like NCCL, never synchronizing a
 * stream, and ranks may share a device). world == 1 is a plain context. */
typedef struct hs_group hs_group;
hs_status hs_group_create(int world, const int* devices, int transport,
                          hs_group** out);
void hs_group_destroy(hs_group* g);
int hs_group_world(const hs_group* g);
int hs_group_transport(const hs_group* g); /* resolved: 0 none, 1 NCCL, 2 in-process */
hs_ctx* hs_group_ctx(hs_group* g, int rank);
/* CG work split of a 2-rank group (SolverConfig::fraction,
 * solver_config.hpp:8-16): rank 0 owns block rows [0, split), rank 1
 * [split, N), split = floor(f N + 0.5) (partition.cpp:11-22) clamped to
 * [1, N-1]; 0 or 1 = the tile-balanced split. Cholesky is 2D block-cyclic. */
hs_status hs_group_set_row_fraction(hs_group* g, double fraction);
hs_status hs_group_set_cholesky_gemm(hs_group* g, int slices);
/* Runs fn(rank, hs_group_ctx(g, rank), arg) on one host thread per rank;
 * returns the first failing rank's status (its message / payload in
 * hs_last_error of the calling thread). */
hs_status hs_group_run(hs_group* g, int (*fn)(int rank, hs_ctx* ctx, void* arg),
                       void* arg);

/* Release what the context keeps between calls: the device matrices cached
 * by the host-buffer entry points (hs_solve_cg_host etc. keep the uploaded
 * matrix), the CG workspace, the Cholesky's INT8 panel buffers and the
 * pinned staging buffers. The next call re-creates what it needs. */
hs_status hs_ctx_trim(hs_ctx* ctx);
int hs_ctx_rank(const hs_ctx* ctx);
int hs_ctx_world(const hs_ctx* ctx);
void* hs_ctx_stream(const hs_ctx* ctx);
/* Number of kernels this library launched on the context so far. */
uint64_t hs_ctx_kernel_launches(const hs_ctx* ctx);
/* Engine of the Cholesky trailing update (gemm_update / syrk_update,
 * block_kernels.cpp:39-57) for later hs_potrf / solve calls on this context:
 * slices = 0 -> FP64 DMMA tensor cores (default, the reference's FP64
 * arithmetic); 1..8 -> FP64 emulated on the INT8 tensor cores (Ozaki scheme,
 * that many 7-bit slices per operand; 8 keeps the worst-case error at the
 * FP64 GEMM rounding bound). Single-GPU and 2D block-cyclic multi-GPU paths,
 * b % 128 == 0; otherwise DMMA. */
hs_status hs_ctx_set_cholesky_gemm(hs_ctx* ctx, int slices);

/* ---- host-side generators (genmat.cpp:16-112, 156-162; exact) ---------- */
uint64_t hs_rng_at(uint64_t key, uint64_t counter);
double hs_rng_uniform_pm1(uint64_t key, uint64_t counter);
hs_status hs_generate_inputs(size_t n, size_t dim, uint64_t seed,
                             double* out /* n*dim */);
double hs_median_pairwise_distance(const double* points, size_t n, size_t dim);
hs_status hs_generate_rhs(size_t n, size_t b, uint64_t seed,
                          double* out /* N*b */);

/* ---- work split (partition.cpp:11-74; host-only, no GPU needed) -------- */
/* split_row = floor(f*N + 0.5)  (partition.hpp:20-22) */
hs_status hs_partition_for_fraction(double fraction, size_t block_rows,
                                    size_t* split_row);
/* beta_j (partition.hpp:24-30) */
hs_status hs_cholesky_border(double fraction, size_t column, size_t block_rows,
                             size_t* beta);
/* Multi-GPU row partition for CG: contiguous block-row ranges balanced by
 * packed-tile count; bounds has world+1 entries (bounds[0]=0,
 * bounds[world]=N). Generalises partition_for_fraction to G devices. */
hs_status hs_partition_rows(size_t block_rows, int world, size_t* bounds);

/* ---- device matrices (BlockedSPDMatrix storage, blocked_matrix.hpp) ---- */
/* Allocates the tiles this rank owns (all tiles when world == 1), zeroed,
 * with identity padding (blocked_matrix.cpp:17-24, 57-74). */
hs_status hs_matrix_create(hs_ctx* ctx, size_t n, size_t b, hs_matrix** out);
/* 2D block-cyclic variant for the distributed Cholesky (hs_potrf on a
 * multi-rank context): tile (i, j) lives on rank (i mod P) * Q + (j mod Q)
 * of a P x Q grid (1x1, 1x2, 2x2, 2x4 for 1/2/4/8 ranks). Same upload /
 * download / assembly semantics (each rank moves only its own tiles). */
hs_status hs_matrix_create_cyclic(hs_ctx* ctx, size_t n, size_t b,
                                  hs_matrix** out);
void hs_matrix_destroy(hs_matrix* m);
hs_status hs_matrix_info(const hs_matrix* m, size_t* n, size_t* b,
                         size_t* row_lo, size_t* row_hi);
/* Full packed array on the host (N(N+1)/2*b*b doubles); a sharded matrix
 * uploads/downloads only its own block rows of it. */
hs_status hs_matrix_upload(hs_matrix* m, const double* host_packed);
hs_status hs_matrix_download(const hs_matrix* m, double* host_packed);
/* dst <- src (same shape and context), device to device. */
hs_status hs_matrix_copy(hs_matrix* dst, const hs_matrix* src);
/* Raw device pointer to the local packed tiles (for tests / interop). */
double* hs_matrix_device_data(hs_matrix* m);

/* ---- (1) GP squared-exponential assembly (genmat.cpp:114-154) ---------- */
/* Device tile generation from host points (n*dim). Element (p,q):
 * p,q >= n -> identity padding; p == q -> sigma_f2 + sigma_n2;
 * else sigma_f2 * exp(-||x_p - x_q||^2 * inv2l2). */
hs_status hs_assemble_se(hs_matrix* m, const double* points, size_t dim,
                         double sigma_f2, double inv2l2, double sigma_n2);
/* generate_spd (genmat.hpp:41-42) without the host matrix: points and the
 * median length-scale rule on the host, tiles on the device. */
hs_status hs_generate_spd(hs_matrix* m, double sigma_f2, double length_scale,
                          double sigma_n2, size_t dim, uint64_t seed);

/* ---- (2) conjugate gradient (cg_solver.hpp:48-49) ---------------------- */
typedef struct {
  double eps;                  /* SolverConfig::eps (solver_config.hpp:13) */
  uint64_t max_iters;          /* SolverConfig::max_iters                   */
  uint64_t recompute_interval; /* SolverConfig::recompute_interval          */
  int record_trace;            /* SolverConfig::record_trace                */
} hs_cg_params;

typedef struct { /* CgStats (cg_solver.hpp:19-29) */
  uint64_t iterations;
  uint64_t recomputations;
  int converged;
  double u0;
  double true_residual; /* ||rhs - A x||_2 at exit */
  double wall_ms;       /* whole call                          */
  double compute_ms;    /* wall minus host<->device transfers  */
  double transfer_ms;   /* H2D/D2H inside the call             */
  int64_t error_iteration;
} hs_cg_stats;

/* Device-resident solve: d_rhs, d_x are N*b device vectors (the rank's full
 * vectors). trace: 3*max_iters host doubles (u, alpha, beta) or NULL. */
hs_status hs_cg_solve(hs_ctx* ctx, const hs_matrix* a, const double* d_rhs,
                      const hs_cg_params* p, double* d_x, hs_cg_stats* stats,
                      double* trace);
/* Drop-in for solve_cg with HOST buffers: uploads the packed matrix and rhs,
 * solves, downloads x (all inside the call, timed as transfer_ms). */
hs_status hs_solve_cg_host(hs_ctx* ctx, size_t n, size_t b,
                           const double* a_packed, const double* rhs,
                           const hs_cg_params* p, double* x,
                           hs_cg_stats* stats, double* trace);

/* t = A x (symv_range over all rows, block_kernels.hpp:34-38). */
hs_status hs_symv(hs_ctx* ctx, const hs_matrix* a, const double* d_x,
                  double* d_y);
/* ||rhs - A x||_2 (the solvers' exit diagnostic). Multi-rank: the matrix
 * must be block-cyclic and x / rhs full-length on every rank (owned-tile
 * partials all-gathered and summed in rank order). */
hs_status hs_true_residual(hs_ctx* ctx, const hs_matrix* a, const double* d_x,
                           const double* d_rhs, double* out);

/* ---- (3) Cholesky (cholesky_solver.hpp:44-58) -------------------------- */
typedef struct {
  double factor_ms;
  double solve_ms;
  double wall_ms;
  double compute_ms;
  double transfer_ms;
  double true_residual;
} hs_chol_stats;

/* In-place factorization: the lower tiles of a hold L (diag-tile upper
 * halves stale). HS_ERR_NOT_SPD with payload (column, pivot);
 * HS_ERR_NUMERICAL on a non-finite factor (cholesky_solver.cpp:222-238). */
hs_status hs_potrf(hs_ctx* ctx, hs_matrix* a, hs_chol_stats* stats);
/* In-place L y = v (forward_substitute) and L^T x = y (back_substitute) on a
 * device vector; HS_ERR_SINGULAR_BLOCK on a zero / NaN diagonal. Multi-rank
 * (block-cyclic L, b % 128 == 0): every rank passes the same full-length v
 * and gets the same result; steps pipeline over tile rows with b-double
 * broadcasts (cholesky_solver.cpp:256-273 semantics). */
hs_status hs_trsv_lower(hs_ctx* ctx, const hs_matrix* l, double* d_v);
hs_status hs_trsv_upper(hs_ctx* ctx, const hs_matrix* l, double* d_v);
/* factorize + substitutions, device resident (a is destroyed, holds L).
 * true_residual needs the original matrix: pass it as a_orig or NULL. */
hs_status hs_solve_spd(hs_ctx* ctx, hs_matrix* a, const double* d_rhs,
                       double* d_x, const hs_matrix* a_orig,
                       hs_chol_stats* stats);
/* Mixed-precision SPD solve with FP64 iterative refinement (the paper's
 * future-work direction; beyond the reference API). The factor
 * of A goes into `work` (same n, b; A stays intact). Its trailing update runs
 * on the INT8 tensor cores with `slices` Ozaki slices (0 = FP64 DMMA).
 * Fewer than 8 slices give a cheaper, less accurate L. Then, in FP64:
 * x = L^-T L^-1 rhs, and per step r = rhs - A x (SYMV over the unmodified
 * A), x += L^-T L^-1 r, until ||r|| <= tol ||rhs||, max_iters steps, or a
 * step that does not halve ||r|| (the FP64 floor of rhs - A x: tol = 0 runs
 * to it). Multi-rank: block-cyclic a and work, full-length vectors on every
 * rank (identical results on every rank, as hs_solve_spd).
 * HS_ERR_NOT_SPD / HS_ERR_NUMERICAL as hs_potrf; a run
 * that ends above tol returns HS_OK with stats->rel_residual > tol. */
typedef struct {
  double factor_ms;
  double solve_ms;  /* first solve + refinement */
  double wall_ms;
  double rel_residual; /* ||rhs - A x|| / ||rhs|| at exit */
  int iterations;      /* refinement steps taken */
  int slices;
} hs_refine_stats;
hs_status hs_solve_spd_refine(hs_ctx* ctx, const hs_matrix* a, hs_matrix* work,
                              const double* d_rhs, double* d_x, int slices,
                              int max_iters, double tol, hs_refine_stats* stats);
/* Drop-ins with HOST buffers (factorize / solve_spd / substitutions). */
hs_status hs_factorize_host(hs_ctx* ctx, size_t n, size_t b, double* a_packed,
                            hs_chol_stats* stats);
hs_status hs_solve_spd_host(hs_ctx* ctx, size_t n, size_t b, double* a_packed,
                            const double* rhs, double* x,
                            hs_chol_stats* stats);
hs_status hs_forward_substitute_host(hs_ctx* ctx, size_t n, size_t b,
                                     const double* l_packed, const double* rhs,
                                     double* y);
hs_status hs_back_substitute_host(hs_ctx* ctx, size_t n, size_t b,
                                  const double* l_packed, const double* y,
                                  double* x);
/* Host-buffer drop-ins over the group (solve_cg / factorize / solve_spd,
 * cg_solver.hpp:48-49, cholesky_solver.hpp:44-58): CG row-sharded (each rank
 * uploads its block rows), Cholesky 2D block-cyclic (each rank moves only its
 * tiles); x is written once. Shapes the distributed kernels do not serve
 * (CG b not in {64,128,256,512}, Cholesky b % 128 != 0) run on rank 0's GPU.
 * The group's ledger is rank 0's (every collective once). */
hs_status hs_group_solve_cg_host(hs_group* g, size_t n, size_t b,
                                 const double* a_packed, const double* rhs,
                                 const hs_cg_params* p, double* x,
                                 hs_cg_stats* stats, double* trace);
hs_status hs_group_factorize_host(hs_group* g, size_t n, size_t b,
                                  double* a_packed, hs_chol_stats* stats);
hs_status hs_group_solve_spd_host(hs_group* g, size_t n, size_t b,
                                  double* a_packed, const double* rhs,
                                  double* x, hs_chol_stats* stats);

/* ---- single-tile kernels (block_kernels.hpp:17-31), for parity tests --- */
/* Batched over `count` independent b x b tiles in device memory. */
hs_status hs_potf_tiles(hs_ctx* ctx, double* d_tiles, size_t b, size_t count,
                        int64_t* first_bad_pivot);
hs_status hs_gemm_update_tiles(hs_ctx* ctx, double* d_c, const double* d_p,
                               const double* d_q, size_t b, size_t count,
                               int lower_only);

/* Kernel-level drop-ins of hsolve::kernels (block_kernels.hpp:16-74), one
 * output element per sequential chain in the reference's order with
 * separately rounded multiply and add (bitwise the reference's results):
 * X_t L_t^T = B_t in place for `count` tiles (trsm_block; singular_block
 * with the first zero / NaN diagonal index as payload b). */
hs_status hs_trsm_tiles(hs_ctx* ctx, double* d_x, const double* d_l, size_t b,
                        size_t count);
/* op 0: potf_block in place (b <= 1024; not_spd payload (-1, pivot) and
 * *bad_pivot); 1: C -= P Q^T (gemm_update); 2: lower(C) -= lower(P P^T)
 * (syrk_update, d_q = d_p). */
hs_status hs_block_exact(hs_ctx* ctx, int op, double* d_c, const double* d_p,
                         const double* d_q, size_t b, int64_t* bad_pivot);
/* y rows of block rows [lo, hi) = (A x) rows, symv_row's order
 * (block_kernels.cpp:59-95) on the packed matrix d_a (N(N+1)/2 b^2). */
hs_status hs_symv_exact(hs_ctx* ctx, const double* d_a, const double* d_x, double* d_y,
                        size_t n, size_t b, size_t lo, size_t hi);
/* op 0: y -= M x (gemv_sub); 1: y -= M^T x (gemv_transpose_sub);
 * 2: L y = y in place (lower_solve); 3: L^T y = y (lower_transpose_solve;
 * singular_block at the first bad row in the solve order) */
hs_status hs_block_vec_op(hs_ctx* ctx, int op, const double* d_m, const double* d_x,
                          double* d_y, size_t b);
/* Block rows [lo, hi) of padded vectors (N*b doubles): op 0: out[i] =
 * row_dot(u, v, i) (one double per row, at index i); 1: out += alpha u
 * (axpy_range); 2: out = u + alpha out (xpay_range); 3: out = u - v
 * (sub_range). */
hs_status hs_range_op(hs_ctx* ctx, int op, double* d_out, const double* d_u,
                      const double* d_v, double alpha, size_t lo, size_t hi, size_t b);

/* C_t -= P_t Q_t^T (t < count) on the INT8 tensor cores with FP64-accurate
 * Ozaki slicing (`slices` int8 slices per operand, 1..8; 8 gives FP64-level
 * error bounds), b % 128 == 0; lower_only as hs_gemm_update_tiles. The
 * emulated-FP64 building block of the Cholesky trailing update (gemm_update /
 * syrk_update, block_kernels.cpp:39-57). */
hs_status hs_oz_gemm_tiles(hs_ctx* ctx, double* d_c, const double* d_p,
                           const double* d_q, size_t b, size_t count,
                           int slices, int lower_only);
/* Tuning hook: later hs_oz_gemm_tiles calls write per-CTA phase timestamps
 * (globaltimer ns; [cta][tile < 64][8]) to this device buffer (NULL: off). */
void hs_oz_set_profile(void* d_buf);

/* ---- profiling hooks (bench.py roofline) ------------------------------- */
/* every > 0: the CG driver brackets every `every`-th SYMV launch with CUDA
 * events on the context stream (0 disables); hs_prof_symv returns
 * (bracketed launches, their total ms). */
void hs_prof_enable(hs_ctx* ctx, int every);
void hs_prof_symv(hs_ctx* ctx, uint64_t* launches, double* total_ms);
void hs_prof_reset(hs_ctx* ctx);

/* ---- communication ledger (transfer_ledger.hpp:9-52) ------------------ */
/* Every NCCL collective a multi-rank context issues is appended to the
 * context's ledger: kind (TransferKind: 0 scalar, 1 subvector, 2 block,
 * 3 block_row, 4 initial_matrix, 5 result), direction (Direction:
 * 2 = bidirectional for collectives), payload bytes (the collective's output
 * buffer on this rank: the full vector for an all-gather, as the reference
 * logs subvector exchanges with the full logical vector,
 * test_cg_solver.cpp:171-176) and step (CG iteration / Cholesky column, -1
 * for setup). Single-GPU contexts issue no collectives, so their ledger stays
 * empty like the reference's homogeneous runs (test_cg_solver.cpp:178-187). */
typedef struct {
  uint8_t kind;
  uint8_t direction;
  uint64_t bytes;
  int64_t step;
} hs_ledger_entry;
size_t hs_ctx_ledger_size(const hs_ctx* ctx);
/* Copies up to `cap` entries (oldest first); returns the number copied. */
size_t hs_ctx_ledger_read(const hs_ctx* ctx, hs_ledger_entry* out, size_t cap);
void hs_ctx_ledger_clear(hs_ctx* ctx);

/* ---- BSPD1 matrix / vector files (matrix_io.hpp:9-19) ------------------- */
/* Format (matrix_io.cpp): "BSPD", version byte 0x01, u64 n, u64 b (little
 * endian), then the packed tiles in triangular order, b*b FP64 row-major per
 * tile. Errors: HS_ERR_IO (cannot open / write), HS_ERR_FORMAT (magic,
 * implausible header n == 0, b == 0, n > 2^32, b > 2^20),
 * HS_ERR_VERSION_MISMATCH (payload expected, actual), HS_ERR_TRUNCATED_FILE
 * (payload expected, actual byte counts). Host-only calls need no GPU. */
hs_status hs_bspd1_probe(const char* path, size_t* n, size_t* b);
hs_status hs_bspd1_read(const char* path, double* host_packed, size_t count);
hs_status hs_bspd1_write(const char* path, size_t n, size_t b,
                         const double* host_packed);
/* Vector files: u64 n then n FP64 values (matrix_io.hpp:16-19). */
hs_status hs_vector_probe(const char* path, size_t* n);
hs_status hs_vector_read(const char* path, double* out, size_t n);
hs_status hs_vector_write(const char* path, size_t n, const double* v);
/* Stream a BSPD1 file straight into device tiles (no host copy of the
 * matrix): pinned staging ring, file reads overlapped with H2D copies. Each
 * rank reads only the tiles it owns (cyclic = 0: its block rows, a contiguous
 * byte range; cyclic = 1: its 2D block-cyclic tiles). Files larger than host
 * RAM load fine. */
hs_status hs_matrix_load_bspd1(hs_ctx* ctx, const char* path, int cyclic,
                               hs_matrix** out);
/* Write a device matrix as BSPD1, streamed through pinned staging. Every rank
 * writes its own tiles at their file offsets (no barrier needed); rank 0
 * writes the header, the rank owning the last block row sets the length. */
hs_status hs_matrix_save_bspd1(const hs_matrix* m, const char* path);

/* ---- diagnostics ------------------------------------------------------ */
/* Read-only HBM bandwidth over `bytes` of device memory, the roofline of the
 * CG SYMV: mode 0 = the SYMV's TMA bulk-copy ring (32-KB slabs, 5 stages,
 * one CTA per SM), mode 1 = plain 128-bit loads, all SMs. Best of `reps`
 * (CUDA events); returns GB/s. */
hs_status hs_probe_hbm_read(hs_ctx* ctx, size_t bytes, int mode, int reps,
                            double* gbs);

#ifdef __cplusplus
}
#endif
#endif /* HS_CUDA_H */
