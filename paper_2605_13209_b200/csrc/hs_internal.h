// Internal types of libhsolve_cuda.so (not part of the ABI).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <vector>

#include "hs_common.cuh"
#include "hs_cuda.h"

namespace hs {

// Lazily dlopen'ed NCCL (only multi-rank contexts need it).
struct Nccl;

// Device scalars of one CG solve (one instance per context).
struct CgScalars {
  double u;       // current r^T r (recurrence value)
  double u0;      // initial r^T r
  double limit;   // eps^2 * u0
  double alpha;
  double beta;
  int64_t iter;   // completed iterations
  int64_t recomputations;
  int32_t done;   // converged / error: later kernels are no-ops
  int32_t status; // HS_OK or HS_ERR_NUMERICAL
  int64_t err_iter;
  uint32_t ticket;  // last-CTA-done counter (reset by the last CTA)
  uint32_t pad;
};

// SYMV work plan: persistent CTAs stream contiguous ranges of 32-KB slabs of
// the packed tiles; partial row / column sums go to fixed segment slots so
// the reduction order is deterministic.
struct SymvPlan {
  int grid = 0;                  // persistent CTAs launched
  int vgrid = 0;                 // work units (dynamically claimed)
  int64_t slabs_per_tile = 0;
  int64_t nrseg = 0;
  // device arrays
  int64_t* cta_slab = nullptr;   // [vgrid+1] slab range per work unit
  int64_t* cta_rseg = nullptr;   // [vgrid] first row segment id
  int64_t* row_rseg = nullptr;   // [own rows+1] row segments of block row i
  int32_t* row_extra = nullptr;  // [row_hi+1]
  int32_t* extra_cta = nullptr;  // [vgrid] units whose first tile is split
  uint32_t* unit_ctr = nullptr;  // next unclaimed unit (reset by finalize)
  double* rowpart = nullptr;     // [nrseg * b]
  double* colmain = nullptr;     // [T_local * b]
  double* colextra = nullptr;    // [vgrid * b]
  // fused CG tail (single rank, hs_cg.cu cg_tail_kernel): balanced items of
  // the per-row partial lists, their sums, tickets, dot / norm partials
  int64_t nitems = 0;
  int tail_grid = 0;             // co-resident CTAs (0: tail kernel unused)
  int4* item = nullptr;          // [nitems] (row, e0, e1, first row segment)
  int2* item_aux = nullptr;      // [nitems] (row segments, first extra)
  int32_t* row_item = nullptr;   // [N + 1]
  double* itempart = nullptr;    // [nitems * b]
  double* tail_dot = nullptr;    // [tail_grid]
  double* tail_rr = nullptr;     // [tail_grid]
  unsigned* tail_bar = nullptr;  // [2]
  // progressive mode (b <= 128, hs_cg.cu): work units walk the block rows
  // from the last to the first, so t_j is complete as soon as block row j is
  // (every tile (k, j) with k >= j has been streamed); a finalizer grid running
  // beside the SYMV sums each row's partials as their block rows complete.
  bool prog = false;
  int4* unit_pos = nullptr;      // [vgrid] (first row, first column, tiles, first row segment)
  int32_t* row_seg0 = nullptr;   // [row_hi] first row segment of block row k
  int32_t* row_nseg = nullptr;   // [row_hi] row segments of block row k (= its arrivals)
  uint32_t* rowdone = nullptr;   // [2][row_hi] arrivals per block row, by launch parity
  uint64_t launch_seq = 0;       // host-side SYMV launch count (parity)
  int64_t* pf = nullptr;         // [2 * pf_units] L2 prefetch (byte offset, bytes) per unit
  int pf_units = 0;
  // two-vector SYMV (CG recompute iterations): the second vector's slots,
  // allocated on first use
  double* rowpart2 = nullptr;    // [nrseg * b]
  double* colmain2 = nullptr;    // [T_local * b]
};

}  // namespace hs

namespace hs {
struct OzPanel;
struct HostStager;
struct LocalComm;  // in-process device-copy collectives (hs_group.cu)
}

struct hs_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  int rank = 0, world = 1;
  hs::Nccl* nccl = nullptr;
  void* comm = nullptr;  // ncclComm_t
  hs_comm_ops ops{};      // custom host transport (hs_ctx_create_custom_comm)
  bool custom = false;
  // rank of a single-process group whose collectives are device copies
  // between the ranks' buffers, ordered by events (hs_group.cu)
  hs::LocalComm* local = nullptr;
  bool distributed() const { return comm != nullptr || custom || local != nullptr; }
  // CG row split of a 2-rank context: fraction of the block rows on rank 0
  // (partition_for_fraction, partition.cpp:11-22); 0 = tile-balanced split
  double row_fraction = 0.0;
  uint64_t launches = 0;
  int num_sms = 148;
  // profiling of the SYMV launches
  bool prof = false;
  int prof_every = 1;        // bracket every k-th SYMV launch with events
  uint64_t prof_counter = 0;
  uint64_t prof_symv_launches = 0;
  double prof_symv_ms = 0.0;
  std::vector<cudaEvent_t> prof_events;  // pairs, drained by hs_prof_symv
  // scratch
  hs::CgScalars* d_scalars = nullptr;
  double* d_dpart = nullptr;  // per-block-row dot partials
  // CG workspace, kept across calls (a cudaMalloc / cudaFree per solve
  // measured 0-80 ms of host stall on a loaded device)
  void* cg_ws = nullptr;
  size_t cg_ws_bytes = 0;
  // small device scratch (status flags), allocated once
  void* scratch = nullptr;
  // general workspaces kept across calls, grown on demand: 0 true residual,
  // 1 distributed Cholesky panels, 2 distributed substitutions, 3 SIMT panels
  void* ws[4] = {nullptr, nullptr, nullptr, nullptr};
  size_t ws_bytes[4] = {0, 0, 0, 0};
  // vectors of the host-buffer entry points, kept across calls
  double* vec[4] = {nullptr, nullptr, nullptr, nullptr};
  size_t vec_cap[4] = {0, 0, 0, 0};
  // INT8-emulation panel buffers of the Cholesky, kept across calls
  hs::OzPanel* oz_panel = nullptr;
  // pinned staging for pageable host buffers (hs_xfer.cu)
  hs::HostStager* stager = nullptr;
  size_t dpart_cap = 0;
  double* h_pinned = nullptr;  // small pinned readback buffer
  // device matrices reused by the host-buffer entry points (slot 0: the
  // solve matrix, slot 1: the unfactored copy kept for the residual)
  // (slots 2, 3: the same for the 2D block-cyclic layout of a multi-rank
  // Cholesky)
  hs_matrix* cache[4] = {nullptr, nullptr, nullptr, nullptr};
  // communication ledger: one entry per NCCL collective (multi-rank only);
  // `step` is the CG iteration / Cholesky column the drivers are in
  std::vector<hs_ledger_entry> ledger;
  int64_t step = -1;
  // Cholesky trailing-update engine: 0 = FP64 DMMA (reference precision),
  // 1..8 = emulated FP64 on the INT8 tensor cores with that many slices
  int chol_slices = 0;
};

struct hs_matrix {
  hs_ctx* ctx = nullptr;
  // layout: 0 = row-sharded (CG; the full matrix when world == 1),
  //         1 = 2D block-cyclic over a P x Q grid (distributed Cholesky)
  int layout = 0;
  int P = 1, Q = 1;
  std::vector<int64_t> owned;      // cyclic: global tile ids held, ascending
  int64_t* d_owned = nullptr;      // cyclic: device copy of `owned`
  std::vector<int64_t> lpos;       // cyclic: global tile -> local slot or -1
  int64_t* d_lpos = nullptr;       // cyclic: device copy of `lpos`
  size_t n = 0, b = 0, N = 0;     // logical size, tile size, block rows
  size_t row_lo = 0, row_hi = 0;  // owned block rows
  int64_t tile_lo = 0, tile_hi = 0;  // owned packed tile range
  double* d = nullptr;            // local tiles
  hs::SymvPlan* plan = nullptr;
  // Cholesky: inverses of the diagonal factor tiles (N * b * b), filled by
  // hs_potrf and reused by the triangular solves.
  double* dinv = nullptr;
  bool has_inv = false;
  // Multi-rank vector layout: row i lives at vec_off[i] (padded rank chunks).
  std::vector<int64_t> bounds;    // world+1 block-row bounds
  int64_t vec_len = 0;            // doubles in a full (padded) vector
  // Multi-rank CG: each rank chunk (vec_len / world doubles) holds its rows
  // (padded to the largest rank) and, from slot_off on, 2 * world doubles of
  // dot-product slots that ride along in the chunk's collectives.
  // slot_off == chunk length when there are no slots.
  int64_t slot_off = 0;
  int64_t* d_row_off = nullptr;   // [N] element offset of block row i
  size_t local_tiles() const {
    return layout == 1 ? owned.size() : (size_t)(tile_hi - tile_lo);
  }
};

namespace hs {

// 2D block-cyclic grid for G ranks: P x Q with P <= Q, P the largest divisor
// of G not above sqrt(G) (1x1, 1x2, 2x2, 2x4, ...); tile (i, j) -> rank
// (i mod P) * Q + (j mod Q).
inline void cyclic_grid(int world, int* P, int* Q) {
  int p = 1;
  for (int d = 1; d * d <= world; ++d)
    if (world % d == 0) p = d;
  *P = p;
  *Q = world / p;
}
inline int cyclic_owner(int64_t i, int64_t j, int P, int Q) {
  return (int)(i % P) * Q + (int)(j % Q);
}

void launch_count(hs_ctx* c, int k = 1);

// ledger kinds (transfer_ledger.hpp:9-16)
enum LedgerKind : uint8_t {
  LK_SCALAR = 0, LK_SUBVECTOR = 1, LK_BLOCK = 2, LK_BLOCK_ROW = 3,
  LK_INITIAL_MATRIX = 4, LK_RESULT = 5
};
// NCCL collectives (hs_ctx.cu); each appends one ledger entry of `kind`
// whose bytes are the collective's output buffer on this rank.
void comm_allgather(hs_ctx* c, const double* send, double* recv, size_t count,
                    LedgerKind kind);
void comm_reduce_scatter(hs_ctx* c, const double* send, double* recv,
                         size_t count, LedgerKind kind);
void comm_bcast_on(hs_ctx* c, const double* send, double* recv, size_t count,
                   int root, cudaStream_t s, LedgerKind kind);
void comm_group(hs_ctx* c, bool start);
void comm_allreduce_max_i64(hs_ctx* c, int64_t* buf, size_t count,
                            cudaStream_t s);
void ensure_plan(hs_matrix* m);
void free_plan(SymvPlan* p);
// y (padded layout, full length) = A x over this rank's tiles (partials of
// other ranks' rows included); dot_out (optional, device) gets per-row dots.
void symv_local(hs_ctx* c, const hs_matrix* m, const double* x, double* y);
// y = A x full-length on every rank (single rank, or block-cyclic over the group)
void symv_full(hs_ctx* c, const hs_matrix* m, const double* x, double* y);
void launch_fill(hs_ctx* c, double* p, double v, int64_t count);
// Scratch matrix of the context for host-buffer calls (created on first use
// or when the shape changes; contents are overwritten by the caller).
hs_matrix* cached_matrix(hs_ctx* c, int slot, size_t n, size_t b);
// In-process group collectives (hs_group.cu): the same contract as the NCCL
// calls they replace, enqueued on stream `s` without blocking the host on
// the GPU (an issue-time rendezvous of the rank threads, then event-ordered
// device copies; peers' buffers are read only after their producers ran).
void local_allgather(hs_ctx* c, const double* send, double* recv, size_t count,
                     cudaStream_t s);
void local_reduce_scatter(hs_ctx* c, const double* send, double* recv, size_t count,
                          cudaStream_t s);
void local_bcast(hs_ctx* c, const double* send, double* recv, size_t count, int root,
                 cudaStream_t s);
void local_allreduce_max_i64(hs_ctx* c, int64_t* buf, size_t count, cudaStream_t s);
void local_comm_release(hs_ctx* c);
void nccl_init_all(hs_ctx** ctxs, int world);
// cuTensorMapEncodeTiled through the runtime's driver entry point (hs_chol.cu):
// `rank`-D map, dims / box in elements, strides (rank-1 of them) in bytes.
CUtensorMap make_tensor_map(CUtensorMapDataType type, const void* base, int rank,
                            const cuuint64_t* dims, const cuuint64_t* strides,
                            const cuuint32_t* box, CUtensorMapSwizzle swizzle);

// Emulated-FP64 (Ozaki, INT8 tensor core) trailing update of the Cholesky
// factorization (hs_oz.cu): int8 slices of a column's panel (single, K = b)
// or of a column pair's joint panel (K = 2b, one exponent per row), each
// double buffered so the next slicing overlaps the current update.
struct OzPanel {
  int b = 0, s = 0;
  int64_t rows = 0;                       // panel rows per buffer ((N-1) b)
  size_t cap_s = 0, cap_sj = 0, cap_e = 0;  // allocated bytes (reused across calls)
  int8_t* S[2] = {nullptr, nullptr};     // [slice][row][K] planes, single column
  int32_t* E[2] = {nullptr, nullptr};    // row exponents
  int8_t* SJ[2] = {nullptr, nullptr};    // column pairs: K = 2b, joint exponents
  int32_t* EJ[2] = {nullptr, nullptr};
  ~OzPanel();
  void init(int b, int64_t N, int s, bool pairs = false);  // reuses big-enough buffers
  void slice(hs_ctx* c, cudaStream_t st, const double* A, int64_t tile_lo, int64_t N,
             int64_t j, const int32_t* status);
  void update(hs_ctx* c, cudaStream_t st, double* A, int64_t tile_lo, int64_t local_tiles,
              int64_t N, int64_t j, bool col, const int32_t* status);
  void slice_pair(hs_ctx* c, cudaStream_t st, const double* A, int64_t tile_lo, int64_t N,
                  int64_t j0, const int32_t* status);
  void update_pair(hs_ctx* c, cudaStream_t st, double* A, int64_t tile_lo, int64_t N,
                   int64_t j0, bool col, int64_t kk, const int32_t* status);
  void slice_contig(hs_ctx* c, cudaStream_t st, const double* X, int64_t N, int64_t j,
                    const int32_t* status);
  void update_list(hs_ctx* c, cudaStream_t st, double* A, const int64_t* lpos, int64_t j,
                   const int32_t* pairs, int64_t npairs, const int32_t* status);
};

// the context's persistent OzPanel / device scratch (lazily allocated)
OzPanel& ctx_oz_panel(hs_ctx* c);
void* ctx_scratch(hs_ctx* c);
// device vector `slot` (0..3) of at least `count` doubles, kept across calls
double* ctx_vec(hs_ctx* c, int slot, size_t count);
// carve `n` buffers of sizes[k] bytes (256-B aligned) out of the context's
// persistent workspace `slot`, growing it when needed
void ctx_workspace(hs_ctx* c, int slot, const size_t* sizes, int n, void** out);
// blocking host <-> device copy of a list of segments: pinned host memory
// goes straight to the DMA engines, pageable memory through the context's
// pinned staging threads (hs_xfer.cu)
struct CopySeg {
  void* dev;
  void* host;
  size_t bytes;
};
void host_copy(hs_ctx* c, const std::vector<CopySeg>& segs, bool h2d);
void free_stager(hs_ctx* c);

}  // namespace hs
