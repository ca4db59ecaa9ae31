// Blocked conjugate gradient on B200 (reference cg_solver.cpp:223-368).
//
// Hot kernel: packed-symmetric SYMV that streams every stored tile of A
// exactly once per matvec. Persistent CTAs (one per SM) claim work units --
// contiguous runs of 32-KB "slabs" (row strips of the row-major tiles),
// guided sizes shrinking towards the end -- from an atomic counter, so CTAs
// on slower SMs simply take fewer units. A producer warp moves slabs + the
// two s-vector segments they need into a 5-stage shared-memory ring with the
// TMA bulk-copy engine (cp.async.bulk + mbarrier complete_tx); 8 consumer
// warps read each element once from shared memory and use it twice: for the
// row sum (A_ij s_j -> t_i) and for the transposed column sum (A_ij^T s_i ->
// t_j). Row sums are accumulated per work unit per block row, column sums
// per tile, into fixed slots that are added in a fixed order, so results
// are deterministic (no atomics on values). Diagonal tiles read only their
// lower triangle (block_kernels.cpp:76-85 semantics).
//
// b <= 128 (the progressive mode, default): the units walk the block rows
// from the last to the first, so t_j is complete as soon as block row j has
// been streamed (every tile (k, j), k >= j, lies in a block row k >= j).
// Consumers announce each finished (unit, block row) segment on a per-row
// counter, and two finalize warps in every CTA add each row's slots while
// the streaming goes on: one launch per matvec, and when the last tile has
// been read only the last block rows' sums remain. b >= 256: memory-order
// walk, then a finalize kernel.
//
// Roofline: HBM-bound. Algorithmic bytes per matvec = packed tile bytes
// (T * b^2 * 8); the partial slots add ~2/b of that (0.8 % at b = 128).
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include <algorithm>
#include <chrono>
#include <cstring>
#include <vector>

#include "hs_internal.h"

namespace hs {


// ---------------------------------------------------------------------------
// CG scalar steps on the device

enum ScalarStep : int { STEP_NONE = 0, STEP_INIT = 1, STEP_ALPHA = 2, STEP_BETA = 3 };

struct StepArgs {
  CgScalars* sc;
  double* trace;       // device trace buffer (3 per iteration) or null
  double eps;
  Dd* dd_slots;        // [world] per-rank partials (multi-GPU) or null
  int world;
  // multi-GPU: the local (hi, lo) partial goes to dd_slots[g * slot_stride]
  // for g < slot_count (one copy per rank chunk of a reduce-scattered
  // buffer); by default to dd_slots[0] only
  int64_t slot_stride = 0;
  int slot_count = 1;
};

// Single-thread scalar step on the combined dot value (cg_solver.cpp lines
// 5, 8-10 and the start-up checks :243-249).
__device__ void scalar_step(int step, double val, const StepArgs& sa) {
  CgScalars* sc = sa.sc;
  if (step == STEP_INIT) {
    sc->u0 = val;
    sc->u = val;
    sc->iter = 0;
    sc->recomputations = 0;
    sc->status = HS_OK;
    sc->err_iter = -1;
    sc->alpha = sc->beta = 0.0;
    if (!isfinite(val)) {
      sc->status = HS_ERR_NUMERICAL;
      sc->err_iter = 0;
      sc->done = 1;
      return;
    }
    sc->limit = sa.eps * sa.eps * val;
    sc->done = (val <= sc->limit) ? 1 : 0;
  } else if (step == STEP_ALPHA) {
    const double alpha = sc->u / val;
    sc->alpha = alpha;
    if (!isfinite(alpha)) {
      sc->status = HS_ERR_NUMERICAL;
      sc->err_iter = sc->iter + 1;
      sc->done = 1;
    }
  } else if (step == STEP_BETA) {
    const double u = val;
    if (!(u >= 0.0) || !isfinite(u)) {
      sc->status = HS_ERR_NUMERICAL;
      sc->err_iter = sc->iter + 1;
      sc->done = 1;
      return;
    }
    const double beta = u / sc->u;
    sc->beta = beta;
    sc->u = u;
    const int64_t it = ++sc->iter;
    if (sa.trace) {
      sa.trace[3 * (it - 1) + 0] = u;
      sa.trace[3 * (it - 1) + 1] = sc->alpha;
      sa.trace[3 * (it - 1) + 2] = beta;
    }
    if (u <= sc->limit) sc->done = 1;
  }
}

// ---------------------------------------------------------------------------
// Fast SYMV for b in {64, 128, 256, 512}

template <int B, int NCW_ = 8, bool PROG_ = false, bool TWO_ = false>
struct SymvCfg {
  // TWO_: two input vectors in one pass over A (t = A s and t2 = A s2; the
  // CG recompute iteration), progressive mode, b <= 128 only
  static constexpr bool TWO = TWO_;
  static constexpr int NCW = NCW_;               // consumer warps
  static constexpr int CT = NCW * 32;            // consumer threads
  // progressive mode: + FW finalize warps (see symv_finalize_rows)
  static constexpr int FW = PROG_ ? 2 : 0;
  static constexpr int THREADS = CT + 32 + FW * 32;  // + one producer warp
  static constexpr int SLAB_BYTES = 32768;
  static constexpr int RS = 4096 / B;    // tile rows per slab
  static constexpr int SPT = B / RS;     // slabs per tile
  static constexpr int TPR = B / 8;      // consumer threads per tile row
  static constexpr int RPP = CT / TPR;   // row lanes
  static constexpr int RT = RS / RPP;    // rows per consumer thread per slab
  static constexpr int W = TPR < 32 ? TPR : 32;  // lanes of a row in a warp
  static constexpr int H = TPR / W;      // warps sharing a row
  // column partials are pre-reduced inside a warp, so one smem row per warp
  // (TPR <= 32) or per row lane (TPR = 64)
  static constexpr int G = TPR <= 32 ? NCW : RPP;
  // 8 consumer warps (16 measured slower: more smem traffic per slab)
  // (6 stages at b <= 128 measured no faster)
  static constexpr int NSTAGE = (B == 512 || TWO_) ? 4 : 5;
  // slab | seg_j (B) | seg_i (RS)
  // (TWO_: a second copy of both segments, staged with every slab)
  static constexpr int SEG_BYTES = (B + RS) * 8 * (TWO_ ? 2 : 1);
  static constexpr int STAGE_BYTES = SLAB_BYTES + SEG_BYTES;
  static constexpr int COLRED_BYTES = G * B * 8;
  static constexpr int YROW_BYTES = H * B * 8;
  // + full/empty mbarriers + per-stage (slab, unit) headers
  static constexpr int SMEM = NSTAGE * STAGE_BYTES + (TWO_ ? 2 : 1) * 2 * COLRED_BYTES +
                              (TWO_ ? 2 * YROW_BYTES : 0) +
                              2 * YROW_BYTES + 2 * NSTAGE * 8 + NSTAGE * 28;
  static_assert(RT >= 1 && RT <= 2 && RS == RT * RPP, "row mapping");
  static_assert(STAGE_BYTES % 16 == 0, "bulk copy alignment");
  static_assert(SMEM <= 227 * 1024, "shared memory budget");
};

struct SymvArgs {
  const double* a;        // local tiles
  const double* s;        // input vector (padded layout)
  const int64_t* row_off; // [N] element offset of block row i in s / out
  int64_t tile_lo;        // global index of the first local tile
  const int64_t* cta_slab;
  const int64_t* cta_rseg;
  double* rowpart;        // [nrseg][B]  (CTA, block row) segments
  double* colmain;        // [T_local][B] column partial of each tile
  double* colextra;       // [grid][B]   a CTA's first tile when it starts
                          //             mid-tile (split tiles)
  const int32_t* done;    // CG early-exit flag (nullable)
  uint32_t* unit_ctr;     // next unclaimed work unit
  int vgrid;              // work units (cta_slab has vgrid + 1 entries)
  unsigned ts_seq;        // launch sequence (HS_SYMV_TIMING builds only)
  // progressive mode (b <= 128; SymvPlan::prog): units from unit_pos walk
  // the block rows downwards, and the end of every (unit, block row) segment
  // is announced by one arrival on rowdone[row] (this launch's parity)
  int prog;
  const int4* unit_pos;
  uint32_t* rowdone;
  // progressive mode: the finalize warps' inputs / outputs
  uint32_t* rowdone_next;   // the other parity's arrivals: reset here
  uint32_t* unit_ctr_next;  // the other parity's unit counter: reset here
  uint32_t* arrivals;       // all segment arrivals of this launch (== nseg: streaming done)
  uint32_t* arrivals_next;  // the other parity's: reset here
  uint32_t nseg;
  const int64_t* pf;        // L2 prefetch of the next launch's unit heads (see plan)
  int pf_units;
  const int32_t* row_seg0;
  const int32_t* row_nseg;
  int64_t row_lo, row_hi;
  double* out;              // t (padded layout)
  const double* dot_s;      // fused dot s . t (or null)
  double* apart;            // [row_hi] per-block-row s . t partials
  int defer;                // 1: leave the partials to the next kernel
  // two-vector mode: the second input, its output and partial slots
  const double* s2;
  double* out2;
  double* rowpart2;
  double* colmain2;
  StepArgs sa;              // otherwise: ticket -> combine -> scalar step / slots
};

__device__ __forceinline__ uint32_t ld_relaxed_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Progressive finalize, run by FW dedicated warps of every SYMV CTA while
// the CTA streams (SymvPlan::prog, b <= 128). The SYMV walks the block rows
// from the last to the first, so t_j -- the row partial(s) of block row j
// plus the column partials of tiles (k, j), k >= j -- is complete as soon as
// block row j has been streamed. The CTA's block rows j = blockIdx.x +
// m * gridDim.x are taken from the highest down; for each, the column
// partials are added in the fixed order k = row_hi - 1 .. max(j, row_lo) as
// the rows k complete (rowdone[k] reaches the row's segment count; 32 rows
// checked per poll, 16 loads in flight), then the row segments of j in claim
// order: deterministic, and when the streaming ends only the partials of
// the last few block rows are still to be added. Each lane owns B / (32 FW)
// columns. s . t is formed per block row (apart[j]); without `defer` the
// last block row to finish (ticket) combines them as a fixed-shape
// double-double tree and applies the scalar step.
template <int B, int FW, bool TWO = false>
__device__ void symv_finalize_rows(const SymvArgs& args, int fw, int lane) {
  constexpr int CPL = B / (32 * FW);  // columns per lane (1 or 2)
  static_assert(CPL == 1 || CPL == 2, "finalize column mapping");
  __shared__ double fin_red[FW];
  __shared__ int fin_last;
  const int col = fw * (B / FW) + lane * CPL;
  const double* colbase = args.colmain - args.tile_lo * B + col;
  // two-vector mode: the second vector's slots, same positions
  const double* colbase2 = TWO ? args.colmain2 - args.tile_lo * B + col : nullptr;
  const int64_t rows = args.row_hi;
  int64_t j = blockIdx.x + ((rows - 1 - blockIdx.x) / gridDim.x) * (int64_t)gridDim.x;
  if (blockIdx.x >= rows) j = -1;
  for (; j >= 0; j -= gridDim.x) {
    double a0 = 0.0, a1 = 0.0, e0 = 0.0, e1 = 0.0;
    int64_t k = rows - 1;
    const int64_t kend = j > args.row_lo ? j : args.row_lo;
    uint64_t t0 = 0;
    while (k >= kend) {
      const int n = (int)(k - kend + 1 < 32 ? k - kend + 1 : 32);
      bool ok = false;
      if (lane < n)
        ok = ld_relaxed_u32(args.rowdone + (k - lane)) == (uint32_t)args.row_nseg[k - lane];
      const unsigned mask = __ballot_sync(0xffffffffu, ok);
      const int ready = mask == 0xffffffffu ? 32 : __ffs(~mask) - 1;
      if (ready == 0) {
        __nanosleep(256);
        // a lost arrival would hang the GPU: fail the launch instead
        uint64_t now;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
        if (t0 == 0) t0 = now;
        else if (now - t0 > 4000000000ull) __trap();
        continue;
      }
      t0 = 0;
      __threadfence();  // acquire: the partials were stored before the arrivals
      int m = 0;
      if constexpr (TWO) {
        // (b = 128 and 64, both vectors; fewer loads in flight per batch)
        for (; m < ready; ++m) {
          const int64_t off = tri(k - m, j) * B;
          if constexpr (CPL == 2) {
            const double2 v = __ldcg(reinterpret_cast<const double2*>(colbase + off));
            const double2 w = __ldcg(reinterpret_cast<const double2*>(colbase2 + off));
            a0 += v.x;
            a1 += v.y;
            e0 += w.x;
            e1 += w.y;
          } else {
            a0 += __ldcg(colbase + off);
            e0 += __ldcg(colbase2 + off);
          }
        }
      } else if constexpr (CPL == 2) {
        for (; m + 16 <= ready; m += 16) {
          double2 v[16];
#pragma unroll
          for (int u = 0; u < 16; ++u)
            v[u] = __ldcg(reinterpret_cast<const double2*>(colbase + tri(k - m - u, j) * B));
#pragma unroll
          for (int u = 0; u < 16; ++u) {
            a0 += v[u].x;
            a1 += v[u].y;
          }
        }
        for (; m < ready; ++m) {
          const double2 v = __ldcg(reinterpret_cast<const double2*>(colbase + tri(k - m, j) * B));
          a0 += v.x;
          a1 += v.y;
        }
      } else {
        for (; m + 16 <= ready; m += 16) {
          double v[16];
#pragma unroll
          for (int u = 0; u < 16; ++u) v[u] = __ldcg(colbase + tri(k - m - u, j) * B);
#pragma unroll
          for (int u = 0; u < 16; ++u) a0 += v[u];
        }
        for (; m < ready; ++m) a0 += __ldcg(colbase + tri(k - m, j) * B);
      }
      k -= ready;
    }
    if (j >= args.row_lo) {
      const int s0 = args.row_seg0[j], ns = args.row_nseg[j];
      for (int e = 0; e < ns; ++e) {
        const double* rp = args.rowpart + (int64_t)(s0 + e) * B + col;
        a0 += __ldcg(rp);
        if (CPL == 2) a1 += __ldcg(rp + 1);
        if constexpr (TWO) {
          const double* rp2 = args.rowpart2 + (int64_t)(s0 + e) * B + col;
          e0 += __ldcg(rp2);
          if (CPL == 2) e1 += __ldcg(rp2 + 1);
        }
      }
    }
    const int64_t o = args.row_off[j] + col;
    args.out[o] = a0;
    if (CPL == 2) args.out[o + 1] = a1;
    if constexpr (TWO) {
      args.out2[o] = e0;
      if (CPL == 2) args.out2[o + 1] = e1;
    }
    if (args.dot_s) {
      double d = args.dot_s[o] * a0;
      if (CPL == 2) d = fma(args.dot_s[o + 1], a1, d);
#pragma unroll
      for (int off = 16; off >= 1; off >>= 1) d += __shfl_xor_sync(0xffffffffu, d, off);
      if (lane == 0) fin_red[fw] = d;
      named_bar_sync(3, FW * 32);
      if (fw == 0 && lane == 0) {
        double pt = fin_red[0];
#pragma unroll
        for (int w = 1; w < FW; ++w) pt += fin_red[w];
        args.apart[j] = pt;
        if (!args.defer) {
          __threadfence();
          fin_last = atomicAdd(&args.sa.sc->ticket, 1u) == (unsigned)rows - 1 ? 1 : 0;
        }
      }
      named_bar_sync(3, FW * 32);
      if (!args.defer && fin_last && fw == 0) {
        // last block row: fixed-shape double-double tree over apart[0..rows)
        __threadfence();
        Dd acc{0.0, 0.0};
        for (int64_t q = lane; q < rows; q += 32) acc = dd_add(acc, __ldcg(args.apart + q));
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1) {
          Dd o2;
          o2.hi = __shfl_xor_sync(0xffffffffu, acc.hi, off);
          o2.lo = __shfl_xor_sync(0xffffffffu, acc.lo, off);
          acc = lane & off ? dd_add(o2, acc) : dd_add(acc, o2);
        }
        if (lane == 0) {
          args.sa.sc->ticket = 0;
          if (args.sa.world == 1) {
            scalar_step(STEP_ALPHA, dd_value(acc), args.sa);
          } else {
            for (int g = 0; g < args.sa.slot_count; ++g)
              args.sa.dd_slots[g * args.sa.slot_stride] = acc;
          }
        }
      }
    }
    if (fw == 0 && lane == 0) args.rowdone_next[j] = 0u;
  }
  if (blockIdx.x == 0 && fw == 0 && lane == 0) {
    *args.unit_ctr_next = 0u;
    *args.arrivals_next = 0u;
  }
}

#ifdef HS_SYMV_TIMING
__device__ unsigned long long g_symv_ts[4096][2];
// finalize per launch: [0] min CTA start (after the PDL wait), [1] max end of
// the partial-slot sums, [2] max CTA end (incl. the dot epilogue)
__device__ unsigned long long g_fin_ts[4096][5];  // + [3] max start, [4] max sums time
// fused tail: [0] min start, [1] max phase-1 end, [2] max barrier-1 exit,
// [3] max phase-2 end, [4] max barrier-2 exit, [5] max end, [6] min barrier-1 exit
__device__ unsigned long long g_tail_ts[4096][7];
// per-CTA stamps of one tail launch (seq == g_tail_cta_seq): start, phase-1
// end, barrier-1 exit, phase-2 end, end
__device__ unsigned long long g_tail_cta[1024][5];
__device__ unsigned g_tail_cta_seq = 100;
__device__ int g_symv_ts_print = 0;
// progressive mode: per launch, the last finalize warp's end
__device__ unsigned long long g_symv_fin_end[4096];
#endif

template <int B, int NCW, bool PROG, bool TWO = false>
__global__ void __launch_bounds__(SymvCfg<B, NCW, PROG, TWO>::THREADS, 1)
    symv_slab_kernel(SymvArgs args) {
  using Cfg = SymvCfg<B, NCW, PROG, TWO>;
  static_assert(!TWO || (PROG && Cfg::SPT <= 4), "two-vector mode: progressive, b <= 128");
  constexpr int RS = Cfg::RS, SPT = Cfg::SPT, TPR = Cfg::TPR, RT = Cfg::RT;
  constexpr int W = Cfg::W, NS = Cfg::NSTAGE, CT = Cfg::CT, G = Cfg::G;

  extern __shared__ __align__(128) unsigned char smem[];
  unsigned char* stages = smem;
  double* colred = reinterpret_cast<double*>(smem + NS * Cfg::STAGE_BYTES);
  double* yrow = colred + 2 * G * B;  // [2][H][B]
  // two-vector mode: the second vector's column / row reduction buffers
  double* colred2 = yrow + 2 * Cfg::H * B;
  double* yrow2 = colred2 + (TWO ? 2 * G * B : 0);
  uint64_t* full = reinterpret_cast<uint64_t*>(yrow2 + (TWO ? 2 * Cfg::H * B : 0));
  uint64_t* empty = full + NS;
  // per-stage header: the slab staged and its work unit (-1: no more work);
  // progressive mode also (block row, column, row end, row segment) of the
  // tile (16-B aligned: 2 * NS mbarriers above)
  int4* hdr_x = reinterpret_cast<int4*>(empty + NS);
  int64_t* hdr_g = reinterpret_cast<int64_t*>(hdr_x + NS);
  int32_t* hdr_u = reinterpret_cast<int32_t*>(hdr_g + NS);

  const int tid = threadIdx.x;
#ifdef HS_SYMV_TIMING
  uint64_t ts_start;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ts_start));
  unsigned sm_id;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(sm_id));
  int64_t ts_slabs = 0;
#endif

  if (tid == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], Cfg::NCW);
    }
    fence_mbar_init();
  }
  for (int k = tid; k < 2 * Cfg::H * B; k += blockDim.x) yrow[k] = 0.0;
  if constexpr (TWO)
    for (int k = tid; k < 2 * Cfg::H * B; k += blockDim.x) yrow2[k] = 0.0;
  __syncthreads();
  // the CTA-private setup above overlaps the previous kernel's tail (PDL);
  // everything below reads its results
  pdl_wait();
  pdl_trigger();
  if (args.done && *args.done) {
    if constexpr (PROG) {
      // a skipped launch still hands the other parity's counters to the
      // next launch (which may run: e.g. the exit residual after CG ends)
      for (int64_t j = blockIdx.x * (int64_t)blockDim.x + tid; j < args.row_hi;
           j += (int64_t)gridDim.x * blockDim.x)
        args.rowdone_next[j] = 0u;
      if (blockIdx.x == 0 && tid == 0) {
        *args.unit_ctr_next = 0u;
        *args.arrivals_next = 0u;
      }
    }
    return;
  }

  if constexpr (PROG) {
    if (tid >= CT + 32) {
      symv_finalize_rows<B, Cfg::FW, TWO>(args, (tid - CT - 32) >> 5, tid & 31);
#ifdef HS_SYMV_TIMING
      if (tid == CT + 32) {
        uint64_t te;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(te));
        atomicMax(&g_symv_fin_end[args.ts_seq % 4096u], (unsigned long long)te);
      }
#endif
      return;
    }
  }
  if (tid >= CT) {
    // ---------------- producer warp ----------------
    // claims work units in order (one atomic per unit) and streams their
    // slabs; the header tells the consumers which slab / unit a stage holds
    if (tid == CT) {
      // A is streamed once per launch: evict-first, so the partial slots the
      // finalize reads next stay in L2
      const uint64_t stream_pol = l2_policy_evict_first();
      // ring position (stage, phase) kept incrementally: a 64-bit % / by NS
      // per slab cost more integer work than the rest of the producer
      int st = 0;
      uint32_t ph = 0;
      bool wrapped = false;  // every stage used once: wait for its release
      if constexpr (PROG) {
        // progressive mode: whole tiles, block rows downwards (row k's
        // tiles j = 0..k in memory order, then row k - 1)
        for (;;) {
          const int u = (int)atomicAdd(args.unit_ctr, 1u);
          if (u >= args.vgrid) {
            if (wrapped) mbar_wait(&empty[st], ph ^ 1u);
            hdr_g[st] = -1;
            hdr_u[st] = -1;
            mbar_arrive(&full[st]);
            // once every segment has arrived (HBM idle until the next
            // SYMV; A is constant over a solve), prefetch into L2 the head of
            // one of the units the next launch's CTAs claim first
            if ((int)blockIdx.x < args.pf_units && args.pf[2 * blockIdx.x + 1] > 0) {
              uint64_t t0 = 0;
              while (ld_relaxed_u32(args.arrivals) != args.nseg) {
                __nanosleep(500);
                uint64_t now;
                asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
                if (t0 == 0) t0 = now;
                else if (now - t0 > 4000000000ull) __trap();
              }
              bulk_prefetch_l2(reinterpret_cast<const unsigned char*>(args.a) + args.pf[2 * blockIdx.x],
                               (uint32_t)args.pf[2 * blockIdx.x + 1]);
            }
            return;
          }
          const int4 up = args.unit_pos[u];
          int64_t k = up.x, j = up.y;
          int seg = up.w;
          for (int n = 0; n < up.z; ++n) {
            const int64_t t = tri(k, j);
            const int rend = (j == k || n + 1 == up.z) ? 1 : 0;
            const int64_t ok = args.row_off[k];
#pragma unroll 1
            for (int q = 0; q < SPT; ++q) {
              if (wrapped) mbar_wait(&empty[st], ph ^ 1u);
              const int64_t g = t * SPT + q;
              hdr_g[st] = g;
              hdr_u[st] = u;
              hdr_x[st] = make_int4((int)k, (int)j, rend, seg);
              unsigned char* buf = stages + st * Cfg::STAGE_BYTES;
              if constexpr (TWO) {
                // both vectors' segments with every slab: slab | s_j | s_i |
                // s2_j | s2_i (the consumers reload s_j per slab)
                mbar_arrive_expect_tx(&full[st], Cfg::SLAB_BYTES + 2 * (B + RS) * 8);
              } else {
                mbar_arrive_expect_tx(&full[st],
                                      Cfg::SLAB_BYTES + RS * 8 + (q == 0 ? B * 8 : 0));
              }
              bulk_g2s_hint(buf, args.a + ((t - args.tile_lo) * B + (int64_t)q * RS) * B,
                            Cfg::SLAB_BYTES, &full[st], stream_pol);
              bulk_g2s(buf + Cfg::SLAB_BYTES + B * 8, args.s + ok + q * RS, RS * 8, &full[st]);
              if (TWO || q == 0)
                bulk_g2s(buf + Cfg::SLAB_BYTES, args.s + args.row_off[j], B * 8, &full[st]);
              if constexpr (TWO) {
                unsigned char* b2 = buf + Cfg::SLAB_BYTES + (B + RS) * 8;
                bulk_g2s(b2, args.s2 + args.row_off[j], B * 8, &full[st]);
                bulk_g2s(b2 + B * 8, args.s2 + ok + q * RS, RS * 8, &full[st]);
              }
              if (++st == NS) {
                st = 0;
                ph ^= 1u;
                wrapped = true;
              }
            }
            if (j == k) {
              --k;
              j = 0;
              ++seg;
            } else {
              ++j;
            }
          }
        }
      } else {
      for (;;) {
        const int u = (int)atomicAdd(args.unit_ctr, 1u);
        if (u >= args.vgrid) {
          if (wrapped) mbar_wait(&empty[st], ph ^ 1u);
          hdr_g[st] = -1;
          hdr_u[st] = -1;
          mbar_arrive(&full[st]);  // end of work, no bytes
          break;
        }
        const int64_t g0 = args.cta_slab[u], g1 = args.cta_slab[u + 1];
        const int64_t t0 = g0 / SPT;
        int64_t t = t0, i = tile_row(t0), j = t0 - tri(tile_row(t0), 0);
        int q = (int)(g0 - t0 * SPT);
        for (int64_t g = g0; g < g1; ++g) {
          if (wrapped) mbar_wait(&empty[st], ph ^ 1u);
          hdr_g[st] = g;
          hdr_u[st] = u;
          unsigned char* buf = stages + st * Cfg::STAGE_BYTES;
          // the s_j (and r_j) segment is constant over a tile: consumers keep
          // it in registers, so it is only staged with a tile's first slab
          const bool seg_j = (q == 0) || (g == g0);
          mbar_arrive_expect_tx(&full[st], Cfg::SLAB_BYTES + RS * 8 + (seg_j ? B * 8 : 0));
          const double* src =
              args.a + ((t - args.tile_lo) * B + (int64_t)q * RS) * B;
          const int64_t oi = args.row_off[i] + q * RS;
          bulk_g2s_hint(buf, src, Cfg::SLAB_BYTES, &full[st], stream_pol);
          bulk_g2s(buf + Cfg::SLAB_BYTES + B * 8, args.s + oi, RS * 8, &full[st]);
          if (seg_j)
            bulk_g2s(buf + Cfg::SLAB_BYTES, args.s + args.row_off[j], B * 8, &full[st]);
          if (++st == NS) {
            st = 0;
            ph ^= 1u;
            wrapped = true;
          }
          if (++q == SPT) {
            q = 0;
            ++t;
            if (++j > i) {
              ++i;
              j = 0;
            }
          }
        }
      }
      }  // memory-order walk
    }
    return;
  }

  // ---------------- consumer warps ----------------
  const int lane = tid & 31, warp = tid >> 5;
  // the partial slots are read by the finalize right after: keep them in L2
  const uint64_t keep_pol = l2_policy_evict_last();
  const int cl = tid % TPR;  // column lane: columns 2cl + 2TPR*m (+1)
  const int rl = tid / TPR;  // row lane: slab rows RT*rl + r
  const int h = cl / W;      // row-sharing warp index (B = 512)
  const int grp = TPR <= 32 ? warp : rl;  // colred row after the warp reduce

  if constexpr (SPT <= 4) {
    // b <= 128: units are whole tiles (ensure_plan), so the loop runs per
    // tile with the slab index q a compile-time constant. A thread's rows
    // recur in every tile of a block row: their partial sums stay in
    // registers (two FMA chains, ra / rb) across the block row and the lanes
    // of a row are reduced once per block row. Fewer instructions per byte
    // matter here: a sustained CG loop runs under the board's power cap.
    static_assert(RT == 2 && Cfg::H == 1 && TPR <= 32, "tiled layout");
    double ra[SPT][RT], rb[SPT][RT], cac[8];
    // two-vector mode: the second vector's row sums (one FMA chain) and
    // column sums
    double r2[SPT][RT], cac2[8];
#pragma unroll
    for (int qq = 0; qq < SPT; ++qq)
#pragma unroll
      for (int r = 0; r < RT; ++r) ra[qq][r] = rb[qq][r] = r2[qq][r] = 0.0;
#pragma unroll
    for (int m = 0; m < 8; ++m) cac[m] = cac2[m] = 0.0;
    double2 sjt[4];
    int cur = -1;
    int64_t ug1 = 0, ti = 0, ii = 0, jj = 0, ifirst = 0, rsg0 = 0;
    int tp = 0, rp = 0;
    int st = 0;  // ring position of the tile's first slab
    uint32_t ph = 0;
    // progressive mode: block row whose finished segment is announced at the
    // next tile end (its stores have drained by then, so the fence is cheap)
    int64_t pend_row = -1;
    for (;;) {
      const int st0 = st;
      mbar_wait(&full[st0], ph);
      const int64_t g = hdr_g[st0];
      if (g < 0) break;
      const int u = hdr_u[st0];
      bool prog_rend = false;
      int64_t prog_seg = 0;
      if constexpr (PROG) {
        const int4 hx = hdr_x[st0];
        ii = hx.x;
        jj = hx.y;
        ti = tri(ii, jj);
        prog_rend = hx.z != 0;
        prog_seg = hx.w;
      } else if (u != cur) {
        cur = u;
        ug1 = args.cta_slab[u + 1];
        ti = args.cta_slab[u] / SPT;
        ii = tile_row(ti);
        jj = ti - tri(ii, 0);
        ifirst = ii;
        rsg0 = args.cta_rseg[u];
      }
#ifdef HS_SYMV_TIMING
      ts_slabs += SPT;
#endif
      if constexpr (!TWO) {
        const double2* sj2 =
            reinterpret_cast<const double2*>(stages + st0 * Cfg::STAGE_BYTES + Cfg::SLAB_BYTES);
#pragma unroll
        for (int m = 0; m < 4; ++m) sjt[m] = sj2[cl + TPR * m];
      }
      const bool diag = ii == jj;
#pragma unroll
      for (int q = 0; q < SPT; ++q) {
        if (q > 0) mbar_wait(&full[st], ph);
        const unsigned char* buf = stages + st * Cfg::STAGE_BYTES;
        const double2* A2 = reinterpret_cast<const double2*>(buf);
        const double2 si2 =
            reinterpret_cast<const double2*>(buf + Cfg::SLAB_BYTES + B * 8)[rl];
        const double sir[2] = {si2.x, si2.y};
        double2 a[RT][4];
#pragma unroll
        for (int r = 0; r < RT; ++r)
#pragma unroll
          for (int m = 0; m < 4; ++m) a[r][m] = A2[(RT * rl + r) * (B / 2) + cl + TPR * m];
        if constexpr (TWO) {
          // both s_j segments come with every slab; the second vector's
          // row and column sums use the same A values
          const double2* sjs = reinterpret_cast<const double2*>(buf + Cfg::SLAB_BYTES);
          const unsigned char* b2 = buf + Cfg::SLAB_BYTES + (B + RS) * 8;
          const double2* sjs2 = reinterpret_cast<const double2*>(b2);
          const double2 si22 = reinterpret_cast<const double2*>(b2 + B * 8)[rl];
          const double sir2[2] = {si22.x, si22.y};
#pragma unroll
          for (int m = 0; m < 4; ++m) sjt[m] = sjs[cl + TPR * m];
#pragma unroll
          for (int r = 0; r < RT; ++r) {
            const int rr = q * RS + RT * rl + r;
#pragma unroll
            for (int m = 0; m < 4; ++m) {
              const double2 sj2 = sjs2[cl + TPR * m];
              const int c0 = 2 * cl + 2 * TPR * m;
              const double ax = a[r][m].x, ay = a[r][m].y;
              // (the diagonal tile: lower triangle only, as below)
              const double rx = !diag || c0 <= rr ? ax : 0.0;
              const double ry = !diag || c0 + 1 <= rr ? ay : 0.0;
              const double cx = !diag || c0 < rr ? ax : 0.0;
              const double cy = !diag || c0 + 1 < rr ? ay : 0.0;
              ra[q][r] = fma(rx, sjt[m].x, ra[q][r]);
              rb[q][r] = fma(ry, sjt[m].y, rb[q][r]);
              cac[2 * m] = fma(cx, sir[r], cac[2 * m]);
              cac[2 * m + 1] = fma(cy, sir[r], cac[2 * m + 1]);
              r2[q][r] = fma(ry, sj2.y, fma(rx, sj2.x, r2[q][r]));
              cac2[2 * m] = fma(cx, sir2[r], cac2[2 * m]);
              cac2[2 * m + 1] = fma(cy, sir2[r], cac2[2 * m + 1]);
            }
          }
        } else if (!diag) {
#pragma unroll
          for (int r = 0; r < RT; ++r)
#pragma unroll
            for (int m = 0; m < 4; ++m) {
              ra[q][r] = fma(a[r][m].x, sjt[m].x, ra[q][r]);
              rb[q][r] = fma(a[r][m].y, sjt[m].y, rb[q][r]);
              cac[2 * m] = fma(a[r][m].x, sir[r], cac[2 * m]);
              cac[2 * m + 1] = fma(a[r][m].y, sir[r], cac[2 * m + 1]);
            }
        } else {
          // diagonal tile: lower triangle only (c <= r for rows, c < r for cols)
#pragma unroll
          for (int r = 0; r < RT; ++r) {
            const int rr = q * RS + RT * rl + r;
#pragma unroll
            for (int m = 0; m < 4; ++m) {
              const int c0 = 2 * cl + 2 * TPR * m;
              ra[q][r] = fma(c0 <= rr ? a[r][m].x : 0.0, sjt[m].x, ra[q][r]);
              rb[q][r] = fma(c0 + 1 <= rr ? a[r][m].y : 0.0, sjt[m].y, rb[q][r]);
              cac[2 * m] = fma(c0 < rr ? a[r][m].x : 0.0, sir[r], cac[2 * m]);
              cac[2 * m + 1] = fma(c0 + 1 < rr ? a[r][m].y : 0.0, sir[r], cac[2 * m + 1]);
            }
          }
        }
        // reads of the stage complete before the TMA refill (hs_chol.cu,
        // gemm_dmma_kernel: ptxas may put the arrive ahead of the last LDS's
        // consumers)
        fence_proxy_async_smem();
        __syncwarp();
        mbar_arrive_if(&empty[st], lane == 0);
        if (++st == NS) {
          st = 0;
          ph ^= 1u;
        }
      }
      // tile end: column partial of tile ti; block row end: row partials
      const bool row_end = PROG ? prog_rend : (diag || (g + SPT == ug1));
      if (row_end) {
#pragma unroll
        for (int qq = 0; qq < SPT; ++qq)
#pragma unroll
          for (int r = 0; r < RT; ++r) {
            double v = ra[qq][r] + rb[qq][r];
#pragma unroll
            for (int off = W / 2; off >= 1; off >>= 1)
              v += __shfl_xor_sync(0xffffffffu, v, off);
            if ((cl & (W - 1)) == 0) yrow[rp * B + qq * RS + RT * rl + r] = v;
            ra[qq][r] = rb[qq][r] = 0.0;
            if constexpr (TWO) {
              double v2 = r2[qq][r];
#pragma unroll
              for (int off = W / 2; off >= 1; off >>= 1)
                v2 += __shfl_xor_sync(0xffffffffu, v2, off);
              if ((cl & (W - 1)) == 0) yrow2[rp * B + qq * RS + RT * rl + r] = v2;
              r2[qq][r] = 0.0;
            }
          }
      }
#pragma unroll
      for (int off = TPR; off < 32; off <<= 1)
#pragma unroll
        for (int m = 0; m < 8; ++m) cac[m] += __shfl_xor_sync(0xffffffffu, cac[m], off);
      double* cr = colred + tp * G * B;
      if (lane < TPR) {
#pragma unroll
        for (int m = 0; m < 4; ++m)
          reinterpret_cast<double2*>(cr + grp * B)[cl + TPR * m] =
              make_double2(cac[2 * m], cac[2 * m + 1]);
      }
      double* cr2 = colred2 + tp * G * B;
      if constexpr (TWO) {
#pragma unroll
        for (int off = TPR; off < 32; off <<= 1)
#pragma unroll
          for (int m = 0; m < 8; ++m) cac2[m] += __shfl_xor_sync(0xffffffffu, cac2[m], off);
        if (lane < TPR) {
#pragma unroll
          for (int m = 0; m < 4; ++m)
            reinterpret_cast<double2*>(cr2 + grp * B)[cl + TPR * m] =
                make_double2(cac2[2 * m], cac2[2 * m + 1]);
        }
      }
      if constexpr (PROG) {
        if (pend_row >= 0 && tid < B) __threadfence();
      }
      named_bar_sync(1, CT);
      if constexpr (PROG) {
        // release pattern: the storing threads fenced before the barrier
        if (pend_row >= 0 && tid == 0) {
          atomicAdd(args.rowdone + pend_row, 1u);
          atomicAdd(args.arrivals, 1u);
        }
        pend_row = -1;
      }
      {
        double* dst = args.colmain + (ti - args.tile_lo) * B;
        for (int c = tid; c < B; c += CT) {
          double acc = 0.0;
#pragma unroll 4
          for (int r = 0; r < G; ++r) acc += cr[r * B + c];
          st_hint(dst + c, acc, keep_pol);
        }
        if constexpr (TWO) {
          double* dst2 = args.colmain2 + (ti - args.tile_lo) * B;
          for (int c = tid; c < B; c += CT) {
            double acc = 0.0;
#pragma unroll 4
            for (int r = 0; r < G; ++r) acc += cr2[r * B + c];
            st_hint(dst2 + c, acc, keep_pol);
          }
        }
      }
      if (row_end) {
        double* yr = yrow + rp * B;
        double* out = args.rowpart + (PROG ? prog_seg : rsg0 + (ii - ifirst)) * B;
        for (int c = tid; c < B; c += CT) st_hint(out + c, yr[c], keep_pol);
        if constexpr (TWO) {
          double* yr2 = yrow2 + rp * B;
          double* o2 = args.rowpart2 + prog_seg * B;
          for (int c = tid; c < B; c += CT) st_hint(o2 + c, yr2[c], keep_pol);
        }
        rp ^= 1;
        // the segment (its column partials and row partial) is announced
        // at the next tile end, or below when the work runs out
        if constexpr (PROG) pend_row = ii;
      }
      tp ^= 1;
#pragma unroll
      for (int m = 0; m < 8; ++m) cac[m] = cac2[m] = 0.0;
      ++ti;
      if (++jj > ii) {
        ++ii;
        jj = 0;
      }
    }
    if constexpr (PROG) {
      if (pend_row >= 0) {
        if (tid < B) __threadfence();
        named_bar_sync(2, CT);
        if (tid == 0) {
          atomicAdd(args.rowdone + pend_row, 1u);
          atomicAdd(args.arrivals, 1u);
        }
      }
    }
  } else {

  double cacc[8];
#pragma unroll
  for (int m = 0; m < 8; ++m) cacc[m] = 0.0;
  double2 sj[4];  // this thread's 8 columns of s_j, kept for the whole tile

  // state of the current work unit (set when its first slab arrives)
  int cur_u = -1;
  int64_t g0 = 0, g1 = 0, t_first = 0, i_first = 0, rseg0 = 0;
  bool split_start = false;
  int64_t t = 0, i = 0, j = 0;
  int q = 0;
  int tpar = 0, rpar = 0;  // parity of tiles / block rows flushed

  int st = 0;  // ring position
  uint32_t ph = 0;
  for (;; st = (st + 1 == NS) ? 0 : st + 1, ph ^= (st == 0) ? 1u : 0u) {
    mbar_wait(&full[st], ph);
    const int64_t g = hdr_g[st];
    if (g < 0) break;
    const int u = hdr_u[st];
    if (u != cur_u) {
      cur_u = u;
      g0 = args.cta_slab[u];
      g1 = args.cta_slab[u + 1];
      t_first = g0 / SPT;
      i_first = tile_row(t_first);
      rseg0 = args.cta_rseg[u];
      split_start = (g0 % SPT) != 0;
      t = t_first;
      i = i_first;
      j = t_first - tri(i_first, 0);
      q = (int)(g0 - t_first * SPT);
    }
#ifdef HS_SYMV_TIMING
    ++ts_slabs;
#endif
    const unsigned char* buf = stages + st * Cfg::STAGE_BYTES;
    const double2* A2 = reinterpret_cast<const double2*>(buf);
    const double* si =
        reinterpret_cast<const double*>(buf + Cfg::SLAB_BYTES + B * 8);

    double2 a[RT][4];
    double sir[RT];
#pragma unroll
    for (int r = 0; r < RT; ++r)
#pragma unroll
      for (int m = 0; m < 4; ++m)
        a[r][m] = A2[(RT * rl + r) * (B / 2) + cl + TPR * m];
    if (q == 0 || g == g0) {  // tile start: load s_j once
      const double2* sj2 =
          reinterpret_cast<const double2*>(buf + Cfg::SLAB_BYTES);
#pragma unroll
      for (int m = 0; m < 4; ++m) sj[m] = sj2[cl + TPR * m];
    }
#pragma unroll
    for (int r = 0; r < RT; ++r) sir[r] = si[RT * rl + r];

    double rs[RT];
#pragma unroll
    for (int r = 0; r < RT; ++r) rs[r] = 0.0;
    // (the stage is released after the FMAs below: an earlier release
    // measured slower)
    if (i != j) {
#pragma unroll
      for (int r = 0; r < RT; ++r) {
        double p0 = 0.0, p1 = 0.0;  // two chains for ILP
#pragma unroll
        for (int m = 0; m < 4; ++m) {
          p0 = fma(a[r][m].x, sj[m].x, p0);
          p1 = fma(a[r][m].y, sj[m].y, p1);
          cacc[2 * m] = fma(a[r][m].x, sir[r], cacc[2 * m]);
          cacc[2 * m + 1] = fma(a[r][m].y, sir[r], cacc[2 * m + 1]);
        }
        rs[r] = p0 + p1;
      }
    } else {
      // diagonal tile: lower triangle only (c <= r for rows, c < r for cols)
#pragma unroll
      for (int r = 0; r < RT; ++r) {
        const int rr = q * RS + RT * rl + r;
        double p0 = 0.0, p1 = 0.0;
#pragma unroll
        for (int m = 0; m < 4; ++m) {
          const int c0 = 2 * cl + 2 * TPR * m;
          p0 = fma(c0 <= rr ? a[r][m].x : 0.0, sj[m].x, p0);
          p1 = fma(c0 + 1 <= rr ? a[r][m].y : 0.0, sj[m].y, p1);
          cacc[2 * m] = fma(c0 < rr ? a[r][m].x : 0.0, sir[r], cacc[2 * m]);
          cacc[2 * m + 1] = fma(c0 + 1 < rr ? a[r][m].y : 0.0, sir[r], cacc[2 * m + 1]);
        }
        rs[r] = p0 + p1;
      }
    }
    fence_proxy_async_smem();  // (see the release in the progressive loop)
    __syncwarp();
    mbar_arrive_if(&empty[st], lane == 0);

    // row sums over the W lanes of a row in this warp; the owning lane adds
    // into yrow[rpar][h][row]
    if (RT == 2) {
      const bool hi = (cl & (W / 2)) != 0;
      const double send = hi ? rs[0] : rs[RT - 1];
      double v = (hi ? rs[RT - 1] : rs[0]) + __shfl_xor_sync(0xffffffffu, send, W / 2);
#pragma unroll
      for (int off = W / 4; off >= 1; off >>= 1)
        v += __shfl_xor_sync(0xffffffffu, v, off);
      if ((cl & (W / 2 - 1)) == 0)
        yrow[(rpar * Cfg::H + h) * B + q * RS + RT * rl + (hi ? 1 : 0)] += v;
    } else {
      double v = rs[0];
#pragma unroll
      for (int off = W / 2; off >= 1; off >>= 1)
        v += __shfl_xor_sync(0xffffffffu, v, off);
      if ((cl & (W - 1)) == 0) yrow[(rpar * Cfg::H + h) * B + q * RS + rl] += v;
    }

    const bool tile_end = (q == SPT - 1) || (g + 1 == g1);
    if (tile_end) {
      const bool row_end = (j == i && q == SPT - 1) || (g + 1 == g1);
      // pre-reduce the row lanes that share columns inside the warp
#pragma unroll
      for (int off = TPR; off < 32; off <<= 1)
#pragma unroll
        for (int m = 0; m < 8; ++m) cacc[m] += __shfl_xor_sync(0xffffffffu, cacc[m], off);
      double* cr = colred + tpar * G * B;
      if (TPR >= 32 || lane < TPR) {
#pragma unroll
        for (int m = 0; m < 4; ++m)
          reinterpret_cast<double2*>(cr + grp * B)[cl + TPR * m] =
              make_double2(cacc[2 * m], cacc[2 * m + 1]);
      }
      named_bar_sync(1, CT);
      double* dst = (split_start && t == t_first)
                        ? args.colextra + (int64_t)u * B
                        : args.colmain + (t - args.tile_lo) * B;
      for (int c = tid; c < B; c += CT) {
        double acc = 0.0;
#pragma unroll 4
        for (int r = 0; r < G; ++r) acc += cr[r * B + c];
        st_hint(dst + c, acc, keep_pol);
      }
      if (row_end) {
        const int64_t rseg = rseg0 + (i - i_first);
        double* yr = yrow + rpar * Cfg::H * B;
        for (int c = tid; c < B; c += CT) {
          double acc = yr[c];
          yr[c] = 0.0;
#pragma unroll
          for (int hh = 1; hh < Cfg::H; ++hh) {
            acc += yr[hh * B + c];
            yr[hh * B + c] = 0.0;
          }
          st_hint(args.rowpart + rseg * B + c, acc, keep_pol);
        }
        rpar ^= 1;
      }
      tpar ^= 1;
#pragma unroll
      for (int m = 0; m < 8; ++m) cacc[m] = 0.0;
    }
    if (++q == SPT) {
      q = 0;
      ++t;
      if (++j > i) {
        ++i;
        j = 0;
      }
    }
  }
  }  // slab-level loop (b >= 256)
#ifdef HS_SYMV_TIMING
  if (tid == 0) {
    uint64_t ts_end;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ts_end));
    if (g_symv_ts_print)
      printf("symvts %d %u %lld %llu %llu\n", blockIdx.x, sm_id, (long long)ts_slabs,
             (unsigned long long)ts_start, (unsigned long long)ts_end);
    // per launch: min start / max end over CTAs (slot = launch sequence)
    const unsigned slot = args.ts_seq % 4096u;
    atomicMin(reinterpret_cast<unsigned long long*>(&g_symv_ts[slot][0]), ts_start);
    atomicMax(reinterpret_cast<unsigned long long*>(&g_symv_ts[slot][1]), ts_end);
  }
#endif
}

// ---------------------------------------------------------------------------
// Finalize: out[row_off[j] + c] = sum of row segments of block row j + sum of
// column segments of tiles (i, j), i >= j, in a fixed order. Optionally
// fused with the per-row dot s_j . out_j and the CG alpha step.

struct Scal;  // fwd

__device__ __forceinline__ double block_sum(double v, double* red) {
  // deterministic fixed-shape tree over the CTA (blockDim multiple of 32)
  for (int off = 16; off >= 1; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  const int w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[w] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0)
    for (int k = 0; k < nw; ++k) s += red[k];
  return s;  // valid in thread 0
}

// Reduce `count` per-CTA partials in fixed order into a double-double.
__device__ Dd dd_reduce_parts(const double* parts, int count, Dd* red) {
  Dd acc{0.0, 0.0};
  for (int k = threadIdx.x; k < count; k += blockDim.x)
    acc = dd_add(acc, parts[k]);
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int w = blockDim.x / 2; w >= 1; w >>= 1) {
    if ((int)threadIdx.x < w) red[threadIdx.x] = dd_add(red[threadIdx.x], red[threadIdx.x + w]);
    __syncthreads();
  }
  return red[0];
}

// Last-CTA epilogue shared by the dot-producing kernels: combine per-CTA
// partials (fixed order); single rank -> apply the scalar step directly,
// multi rank -> publish this rank's (hi, lo) for the all-gather.
__device__ void dot_epilogue(double part, double* dpart, int slot, int count,
                             int step, const StepArgs& sa) {
  __shared__ double red_d[32];
  __shared__ Dd red_dd[256];  // up to 256 threads (finalize, vector kernels)
  __shared__ bool last;
  const double p = block_sum(part, red_d);
  if (threadIdx.x == 0) {
    dpart[slot] = p;
    __threadfence();
    const unsigned prev = atomicAdd(&sa.sc->ticket, 1u);
    last = (prev == (unsigned)count - 1);
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  const Dd tot = dd_reduce_parts(dpart, count, red_dd);
  if (threadIdx.x == 0) {
    sa.sc->ticket = 0;
    if (sa.world == 1) {
      scalar_step(step, dd_value(tot), sa);
    } else {
      // local partial, carried to the other ranks by the host driver's
      // collective (all-gather, or inside the reduce-scatter of t)
      for (int g = 0; g < sa.slot_count; ++g) sa.dd_slots[g * sa.slot_stride] = tot;
    }
  }
}

struct FinalizeArgs {
  const int64_t* row_rseg;   // [own rows+1] row segments
  const int32_t* row_extra;  // [rows+1] range into extra_cta
  const int32_t* extra_cta;  // units whose first (split) tile is in column j
  const double* rowpart;
  const double* colmain;
  const double* colextra;
  uint32_t* unit_ctr;        // SYMV work-unit counter, reset here
  unsigned ts_seq;           // launch sequence (HS_SYMV_TIMING builds only)
  const int64_t* row_off;
  int64_t row_lo, row_hi, tile_lo;
  int b;
  double* out;         // padded layout
  const double* s;     // for the fused dot (padded layout) or null
  double* dpart;
  double* apart;       // deferred alpha: per-CTA s.t partials only (see V_UPDATE)
  int step;
  StepArgs sa;
  const int32_t* done;
  // L2 prefetch of the next SYMV's first slabs (see finalize_kernel)
  const unsigned char* pf_base;  // local tiles (bytes)
  const int64_t* pf_slab;        // the plan's cta_slab
  int64_t pf_slab_lo;            // global index of the first local slab
  int pf_units;                  // units claimed first (one per SYMV CTA)
  int pf_slabs;                  // slabs prefetched per unit (0: off)
};

// Block row j (blockIdx.x), 32 columns (blockIdx.y): out_j[c] is the sum of
// every partial b-vector that lands on block row j -- the column partials
// of tiles (i, j), the row segments of the units that covered row j, and the
// split-tile extras. The FIN_WARPS warps of the CTA take the partials
// round-robin (one coalesced 256-B load per warp per partial, 8 loads in
// flight per thread), then warp 0 adds the per-warp sums in a fixed order:
// deterministic. Small CTAs so the whole grid (N * b / 32 CTAs) is resident
// in one wave. Optionally fused with the dot s_j . out_j and, via a global
// ticket, the alpha step.
constexpr int FIN_WARPS = 8;
constexpr int FIN_THREADS = FIN_WARPS * 32;
constexpr int FIN_COLS = 32;

// (8 CTAs per SM: the whole N * b / 32 grid must be resident in one wave)
__global__ void __launch_bounds__(FIN_THREADS, 8) finalize_kernel(FinalizeArgs fa) {
  const int64_t jr = blockIdx.x;  // output block row
  const int b = fa.b;
  const int cl = threadIdx.x & 31, p = threadIdx.x >> 5;
  const int c = blockIdx.y * FIN_COLS + cl;
  __shared__ double red[FIN_WARPS][33];
  // entries: [0, nc) column partials of tiles (i0 + e, jr); [nc, nc + nrs)
  // row segments; then the split-tile extras
  const int64_t i0 = jr > fa.row_lo ? jr : fa.row_lo;
  const int64_t nc = fa.row_hi - i0;
  const bool own = jr >= fa.row_lo && jr < fa.row_hi;
  const int64_t rs0 = own ? fa.row_rseg[jr - fa.row_lo] : 0;
  const int64_t nrs = own ? fa.row_rseg[jr - fa.row_lo + 1] - rs0 : 0;
  const int e0 = fa.row_extra[jr];
  const int64_t ne = fa.row_extra[jr + 1] - e0;
  const int64_t E = nc + nrs + ne;
  const double* colbase = fa.colmain - fa.tile_lo * b + c;
  const int64_t o = fa.row_off[jr] + c;
  // the plan lookups above overlap the SYMV's tail (PDL); the partial slots
  // below are its output
  pdl_wait();
  pdl_trigger();
#ifdef HS_SYMV_TIMING
  unsigned long long ft0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ft0));
#endif
  if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) *fa.unit_ctr = 0u;
  if (fa.done && *fa.done) return;
  {
    // HBM is nearly idle from here to the next SYMV (the partial slots below
    // are L2 hits): prefetch into L2 the first slabs of the units the next
    // SYMV's CTAs claim first (units 0 .. grid-1; A is constant over the
    // solve), so its ramp-up reads hit L2 instead of waiting on HBM
    const int lin = (int)(blockIdx.x * gridDim.y + blockIdx.y);
    if (lin < fa.pf_units && threadIdx.x == 0) {
      const int64_t g0 = fa.pf_slab[lin], g1 = fa.pf_slab[lin + 1];
      const int64_t ns = g1 - g0 < fa.pf_slabs ? g1 - g0 : fa.pf_slabs;
      if (ns > 0)
        bulk_prefetch_l2(fa.pf_base + (g0 - fa.pf_slab_lo) * 32768, (uint32_t)(ns * 32768));
    }
  }
  // entries e = p, p + FIN_WARPS, ... added in that order. The column
  // partials (a heavy row has ~N of them) are loaded 8 at a time before the
  // adds, so the loads overlap instead of forming a serial chain (the plain
  // `acc += load` loop measured 18 us for the heaviest row)
  double acc = 0.0;
  int64_t e = p;
  for (; e + 7 * FIN_WARPS < nc; e += 8 * FIN_WARPS) {
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = __ldg(colbase + tri(i0 + e + u * FIN_WARPS, jr) * b);
#pragma unroll
    for (int u = 0; u < 8; ++u) acc += v[u];
  }
  for (; e < nc; e += FIN_WARPS) acc += __ldg(colbase + tri(i0 + e, jr) * b);
#pragma unroll 4
  for (; e < nc + nrs; e += FIN_WARPS) acc += __ldg(fa.rowpart + (rs0 + e - nc) * b + c);
  for (; e < E; e += FIN_WARPS)
    acc += __ldg(fa.colextra + (int64_t)fa.extra_cta[e0 + (e - nc - nrs)] * b + c);
  red[p][cl] = acc;
  __syncthreads();
  double dotp = 0.0;
  if (p == 0) {
    double t = 0.0;
#pragma unroll
    for (int pp = 0; pp < FIN_WARPS; ++pp) t += red[pp][cl];
    fa.out[o] = t;
    if (fa.s) dotp = fa.s[o] * t;
  }
#ifdef HS_SYMV_TIMING
  unsigned long long ft1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ft1));
#endif
  if (fa.apart) {
    // deferred alpha: the per-CTA partial only; the next vector kernel's
    // CTAs reduce the partials themselves (no ticket, no last-CTA tail)
    __shared__ double red_d[32];
    const double pt = block_sum(dotp, red_d);
    if (threadIdx.x == 0) fa.apart[jr * gridDim.y + blockIdx.y] = pt;
  } else if (fa.s) {
    dot_epilogue(dotp, fa.dpart, (int)(jr * gridDim.y + blockIdx.y),
                 (int)(gridDim.x * gridDim.y), fa.step, fa.sa);
  }
#ifdef HS_SYMV_TIMING
  if (threadIdx.x == 0) {
    unsigned long long ft2;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ft2));
    const unsigned sl = fa.ts_seq % 4096u;
    atomicMin(&g_fin_ts[sl][0], ft0);
    atomicMax(&g_fin_ts[sl][1], ft1);
    atomicMax(&g_fin_ts[sl][2], ft2);
    atomicMax(&g_fin_ts[sl][3], ft0);
    atomicMax(&g_fin_ts[sl][4], ft1 - ft0);
  }
#endif
}

// ---------------------------------------------------------------------------
// Generic SYMV (any b; single rank): one warp per output row reading the
// packed symmetric storage like symv_row (block_kernels.cpp:59-95).

__global__ void symv_generic_kernel(const double* __restrict__ a, int64_t n_pad,
                                    int b, const double* __restrict__ x,
                                    double* __restrict__ y,
                                    const int32_t* done) {
  pdl_wait();
  pdl_trigger();
  if (done && *done) return;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= n_pad) return;
  const int64_t p = warp;
  const int64_t ip = p / b;
  const int r = (int)(p - ip * b);
  double acc = 0.0;
  for (int64_t qq = lane; qq < n_pad; qq += 32) {
    const int64_t iq = qq / b;
    const int c = (int)(qq - iq * b);
    double v;
    if (iq < ip || (iq == ip && c <= r))
      v = a[tri(ip, iq) * b * b + (int64_t)r * b + c];
    else
      v = a[tri(iq, ip) * b * b + (int64_t)c * b + r];
    acc = fma(v, x[qq], acc);
  }
  for (int off = 16; off >= 1; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
  if (lane == 0) y[p] = acc;
}

// ---------------------------------------------------------------------------
// Vector kernels over a rank's local chunk (len elements). Every kernel that
// produces a dot uses a fixed grid and a fixed per-thread element set, so the
// reduction order is deterministic.

constexpr int VGRID = 148;
constexpr int VBLOCK = 256;

struct VecArgs {
  int64_t len;
  double* x;
  double* r;
  double* s;        // local chunk of s
  const double* t;
  const double* rhs;
  double* dpart;
  StepArgs sa;
  const int32_t* done;
  int mode;
  // V_UPDATE with a deferred alpha: the finalize's per-CTA s.t partials
  // (reduced here by every CTA in the finalize's fixed order)
  const double* apart = nullptr;
  int acount = 0;
  const double* t2 = nullptr;  // V_RECOMP: A x_old
};

enum VecMode : int {
  V_INIT = 0,       // x = 0, r = s = rhs, dot(rhs, rhs) -> INIT
  V_UPDATE = 1,     // x += a s, r -= a t, dot(r, r) -> BETA
  V_AXPY_X = 2,     // x += a s (recompute iteration, first half)
  V_RESIDUAL = 3,   // r = rhs - t, dot(r, r) -> BETA (recompute second half)
  V_SDIR = 4,       // s = r + beta s
  V_DOT_ST = 5,     // dot(s, t) -> ALPHA (after the generic SYMV)
  V_RESNORM = 6,    // dot(rhs - t, rhs - t) -> NONE (true residual)
  // recompute iteration from one two-vector pass (t = A s, t2 = A x_old):
  // x += a s, r = rhs - (t2 + a t) = rhs - A x_new, dot(r, r) -> BETA
  V_RECOMP = 7,
};

__global__ void __launch_bounds__(VBLOCK) vec_kernel(VecArgs va) {
  pdl_wait();
  pdl_trigger();
  if (va.mode != V_INIT && va.mode != V_RESNORM && va.done && *va.done) return;
  double alpha = va.sa.sc->alpha;
  const double beta = va.sa.sc->beta;
  if (va.apart) {
    // alpha = u / s^T t from the finalize's partials: every CTA computes the
    // same double-double sum (same order and tree shape as the finalize's
    // own last-CTA reduction); CTA 0 keeps the books (alpha, non-finite ->
    // done / status). A non-finite alpha skips the update, as `done` would.
    __shared__ Dd red_a[VBLOCK];
    const double st = dd_value(dd_reduce_parts(va.apart, va.acount, red_a));
    alpha = va.sa.sc->u / st;
    if (blockIdx.x == 0 && threadIdx.x == 0) scalar_step(STEP_ALPHA, st, va.sa);
    if (!isfinite(alpha)) return;
  }
  double part = 0.0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < va.len;
       k += stride) {
    switch (va.mode) {
      case V_INIT: {
        const double v = va.rhs[k];
        va.x[k] = 0.0;
        va.r[k] = v;
        va.s[k] = v;
        part = fma(v, v, part);
        break;
      }
      case V_UPDATE: {
        va.x[k] = fma(alpha, va.s[k], va.x[k]);
        const double rr = fma(-alpha, va.t[k], va.r[k]);
        va.r[k] = rr;
        part = fma(rr, rr, part);
        break;
      }
      case V_AXPY_X:
        va.x[k] = fma(alpha, va.s[k], va.x[k]);
        break;
      case V_RESIDUAL: {
        const double rr = va.rhs[k] - va.t[k];
        va.r[k] = rr;
        part = fma(rr, rr, part);
        break;
      }
      case V_SDIR:
        va.s[k] = fma(beta, va.s[k], va.r[k]);
        break;
      case V_DOT_ST:
        part = fma(va.s[k], va.t[k], part);
        break;
      case V_RESNORM: {
        const double rr = va.rhs[k] - va.t[k];
        part = fma(rr, rr, part);
        break;
      }
      case V_RECOMP: {
        va.x[k] = fma(alpha, va.s[k], va.x[k]);
        const double rr = va.rhs[k] - fma(alpha, va.t[k], va.t2[k]);
        va.r[k] = rr;
        part = fma(rr, rr, part);
        break;
      }
    }
  }
  int step = STEP_NONE;
  if (va.mode == V_INIT) step = STEP_INIT;
  else if (va.mode == V_UPDATE || va.mode == V_RESIDUAL || va.mode == V_RECOMP) step = STEP_BETA;
  else if (va.mode == V_DOT_ST) step = STEP_ALPHA;
  else if (va.mode == V_RESNORM) step = STEP_NONE;
  else return;
  dot_epilogue(part, va.dpart, blockIdx.x, gridDim.x, step, va.sa);
}

// Combine all-gathered per-rank (hi, lo) partials in rank order, then the
// scalar step (multi-rank path; identical on every rank).
__global__ void combine_kernel(const Dd* slots, int64_t stride, int world, int step,
                               StepArgs sa, double* out_value,
                               const int32_t* done) {
  if (step != STEP_INIT && step != STEP_NONE && done && *done) return;
  Dd acc = slots[0];
  for (int g = 1; g < world; ++g) acc = dd_add(acc, slots[g * stride]);
  const double v = dd_value(acc);
  if (out_value) *out_value = v;
  if (step != STEP_NONE) scalar_step(step, v, sa);
}

// ---------------------------------------------------------------------------
// Fused CG tail (single GPU, plain iterations): everything between two SYMVs
// in ONE kernel -- t from the partial slots, alpha, x / r updates, r^T r,
// beta, s = r + beta s (cg_solver.cpp:258-332) -- instead of finalize +
// update + direction (three launches, two of them short latency-bound vector
// kernels, and a finalize set by the heaviest block row's ~N column
// partials). Persistent co-resident grid (cooperative launch), two grid
// barriers, no other inter-CTA waits:
//   phase 1: the finalize's partial sums, balanced: block row j's entry list
//     (column partials of tiles (j..N-1, j), its row segments, split-tile
//     extras; the finalize's order) is cut into items of at most TAIL_ITEM
//     entries; one warp per (item, 32 columns) sums its entries (16 loads in
//     flight) into an item partial, and accumulates s_j . (item partial) --
//     s . t is linear in the partials, so no combine is needed for alpha.
//     Per-CTA s . t partial (fixed order over the CTA's warps and units).
//   barrier; every CTA reduces the s . t partials in one fixed order
//     (identical alpha everywhere); per element, t = the row's item partials
//     added in item order; x += alpha s, r -= alpha t; r . r partial per CTA.
//   barrier; every CTA reduces the r . r partials -> beta; s = r + beta s.
// CTA 0 keeps the scalar books (scalar_step: alpha / beta, non-finite
// checks, trace, done). Deterministic: every sum has a fixed order and shape
// for a given grid (the grid is fixed per device).
constexpr int TAIL_THREADS = 256;
constexpr int TAIL_ITEM = 32;   // entries per item
constexpr int TAIL_BATCH = 16;  // loads in flight per lane

struct TailArgs {
  const double* rowpart;
  const double* colmain;
  const double* colextra;
  const int32_t* extra_cta;
  uint32_t* unit_ctr;
  int64_t N;
  int b, nch, lgb;             // b = 1 << lgb
  const int4* item;            // [nitems] (row j, e0, e1, first row segment)
  const int2* item_aux;        // [nitems] (row segments of j, first extra of j)
  const int32_t* row_item;     // [N + 1]
  int64_t nitems;
  double* itempart;            // [nitems * b]
  double* dotpart;             // [grid]
  double* rrpart;              // [grid]
  unsigned* bar;               // [2] grid-barrier counters
  int64_t len;                 // N * b
  double* x;
  double* r;
  double* s;
  StepArgs sa;
  const int32_t* done;
  const unsigned char* pf_base;
  const int64_t* pf_slab;
  int64_t pf_slab_lo;
  int pf_units, pf_slabs;
  unsigned ts_seq;  // launch sequence (HS_SYMV_TIMING builds only)
};

#ifdef HS_SYMV_TIMING
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define TAIL_TS(k, op)                                                        \
  if (threadIdx.x == 0) atomic##op(&g_tail_ts[ta.ts_seq % 4096u][k], gtime());
#define TAIL_CTA(k)                                                           \
  if (threadIdx.x == 0 && ta.ts_seq == g_tail_cta_seq && blockIdx.x < 1024)    \
    g_tail_cta[blockIdx.x][k] = gtime();
#else
#define TAIL_TS(k, op)
#define TAIL_CTA(k)
#endif

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// all CTAs of a co-resident grid; writes before it are visible after it
__device__ __forceinline__ void tail_grid_barrier(unsigned* ctr) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(ctr, 1u);
    while (ld_acquire_u32(ctr) < gridDim.x) {
    }
  }
  __syncthreads();
}

// fixed-order double-double sum of `count` values read through L2 (written
// by other CTAs of this grid before a barrier)
__device__ Dd dd_reduce_cg(const double* parts, int64_t count, Dd* red) {
  Dd acc{0.0, 0.0};
  for (int64_t k = threadIdx.x; k < count; k += blockDim.x) acc = dd_add(acc, __ldcg(parts + k));
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int w = blockDim.x / 2; w >= 1; w >>= 1) {
    if ((int)threadIdx.x < w) red[threadIdx.x] = dd_add(red[threadIdx.x], red[threadIdx.x + w]);
    __syncthreads();
  }
  const Dd out = red[0];
  __syncthreads();
  return out;
}

__global__ void __launch_bounds__(TAIL_THREADS, 4) cg_tail_kernel(TailArgs ta) {
  pdl_wait();
  if (ta.done && *ta.done) return;
  TAIL_TS(0, Min)
  TAIL_CTA(0)
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int b = ta.b, nch = ta.nch;
  const int64_t N = ta.N;
  const double u_old = ta.sa.sc->u;  // CTA 0 replaces it after barrier 2
  __shared__ double red_w[TAIL_THREADS / 32];
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    ta.bar[1] = 0u;      // nobody reaches barrier 2 before CTA 0 arrives at barrier 1
    *ta.unit_ctr = 0u;   // SYMV work-unit counter for the next launch
  }
  // ---- phase 1: item partials and s . t ----
  const int64_t gwarp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t units = ta.nitems * nch;
  double dacc = 0.0;
  for (int64_t u = gwarp; u < units; u += nwarps) {
    const int64_t it = u / nch;
    const int ch = (int)(u - it * nch);
    const int4 d = __ldg(ta.item + it);
    const int64_t j = d.x, e1 = d.z;
    const int c = ch * 32 + lane;
    const double sj = ta.s[(j << ta.lgb) + c];
    const int64_t nc = N - j;  // column partials of tiles (j .. N-1, j)
    const double* colbase = ta.colmain + c;
    double acc = 0.0;
    int64_t e = d.y;
    // column partials in predicated batches: every load of a batch is in
    // flight at once (a scalar remainder loop is one L2 round trip per
    // entry); the absent entries add exact zeros
    const int64_t ce = e1 < nc ? e1 : nc;
    if (e < ce) {
      for (; e < ce; e += TAIL_BATCH) {
        double v[TAIL_BATCH];
#pragma unroll
        for (int k = 0; k < TAIL_BATCH; ++k)
          v[k] = e + k < ce ? __ldg(colbase + (tri(j + e + k, j) << ta.lgb)) : 0.0;
#pragma unroll
        for (int k = 0; k < TAIL_BATCH; ++k) acc += v[k];
      }
      e = ce;
    }
    if (e < e1) {  // row segments, then split-tile extras
      const int2 a = __ldg(ta.item_aux + it);
      for (; e < e1 && e < nc + a.x; ++e) acc += __ldg(ta.rowpart + ((d.w + e - nc) << ta.lgb) + c);
      for (; e < e1; ++e)
        acc += __ldg(ta.colextra + ((int64_t)ta.extra_cta[a.y + (e - nc - a.x)] << ta.lgb) + c);
    }
    ta.itempart[(it << ta.lgb) + c] = acc;
    dacc = fma(sj, acc, dacc);
  }
  for (int off = 16; off >= 1; off >>= 1) dacc += __shfl_xor_sync(0xffffffffu, dacc, off);
  if (lane == 0) red_w[warp] = dacc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
#pragma unroll
    for (int w = 0; w < TAIL_THREADS / 32; ++w) t += red_w[w];
    ta.dotpart[blockIdx.x] = t;
  }
  TAIL_TS(1, Max)
  TAIL_CTA(1)
  tail_grid_barrier(&ta.bar[0]);
  TAIL_TS(2, Max)
  TAIL_CTA(2)
  TAIL_TS(6, Min)
  pdl_trigger();  // every tail CTA is resident: the next SYMV may launch
  if ((int)blockIdx.x < ta.pf_units && threadIdx.x == 0 && ta.pf_slabs > 0) {
    // L2 prefetch of the next SYMV's first slabs (as finalize_kernel), after
    // phase 1 so the fills do not compete with the partial-slot reads
    const int64_t g0 = ta.pf_slab[blockIdx.x], g1 = ta.pf_slab[blockIdx.x + 1];
    const int64_t ns = g1 - g0 < ta.pf_slabs ? g1 - g0 : ta.pf_slabs;
    if (ns > 0)
      bulk_prefetch_l2(ta.pf_base + (g0 - ta.pf_slab_lo) * 32768, (uint32_t)(ns * 32768));
  }
  // ---- phase 2: alpha; t; x, r; r . r ----
  __shared__ Dd red[TAIL_THREADS];
  __shared__ double red_d[32];
  const double st = dd_value(dd_reduce_cg(ta.dotpart, gridDim.x, red));
  const double alpha = u_old / st;
  if (blockIdx.x == 0 && threadIdx.x == 0) scalar_step(STEP_ALPHA, st, ta.sa);
  if (!isfinite(alpha)) {
    if (blockIdx.x == 0 && threadIdx.x == 0) ta.bar[0] = 0u;  // all passed barrier 1
    return;
  }
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  double part = 0.0;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < ta.len; k += stride) {
    const int64_t j = k >> ta.lgb;
    const int c = (int)(k & (b - 1));
    const int i0 = __ldg(ta.row_item + j), m = __ldg(ta.row_item + j + 1) - i0;
    double t = 0.0;
    for (int q0 = 0; q0 < m; q0 += 8) {  // predicated batches, as in phase 1
      double v[8];
#pragma unroll
      for (int q = 0; q < 8; ++q)
        v[q] = q0 + q < m ? __ldcg(ta.itempart + ((int64_t)(i0 + q0 + q) << ta.lgb) + c) : 0.0;
#pragma unroll
      for (int q = 0; q < 8; ++q) t += v[q];
    }
    ta.x[k] = fma(alpha, ta.s[k], ta.x[k]);
    const double rr = fma(-alpha, t, ta.r[k]);
    ta.r[k] = rr;
    part = fma(rr, rr, part);
  }
  const double pc = block_sum(part, red_d);
  if (threadIdx.x == 0) ta.rrpart[blockIdx.x] = pc;
  TAIL_TS(3, Max)
  TAIL_CTA(3)
  tail_grid_barrier(&ta.bar[1]);
  TAIL_TS(4, Max)
  // ---- phase 3: beta; s = r + beta s ----
  const double un = dd_value(dd_reduce_cg(ta.rrpart, gridDim.x, red));
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    scalar_step(STEP_BETA, un, ta.sa);
    ta.bar[0] = 0u;  // every CTA passed barrier 1
  }
  if (!(un >= 0.0) || !isfinite(un)) return;
  const double beta = un / u_old;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < ta.len; k += stride)
    ta.s[k] = fma(beta, ta.s[k], ta.r[k]);
  __syncthreads();
  TAIL_TS(5, Max)
  TAIL_CTA(4)
}

// ---------------------------------------------------------------------------
// plan

void free_plan(SymvPlan* p) {
  if (!p) return;
  for (void* q : {(void*)p->cta_slab, (void*)p->cta_rseg, (void*)p->row_rseg,
                  (void*)p->row_extra, (void*)p->extra_cta, (void*)p->unit_ctr,
                  (void*)p->rowpart, (void*)p->colmain, (void*)p->colextra,
                  (void*)p->item, (void*)p->item_aux, (void*)p->row_item,
                  (void*)p->itempart, (void*)p->tail_dot, (void*)p->tail_rr,
                  (void*)p->tail_bar, (void*)p->unit_pos, (void*)p->row_seg0,
                  (void*)p->row_nseg, (void*)p->rowdone, (void*)p->pf,
                  (void*)p->rowpart2, (void*)p->colmain2})
    cudaFree(q);
  delete p;
}

static bool fast_b(size_t b) { return b == 64 || b == 128 || b == 256 || b == 512; }

template <typename T>
static void upload_vec(T** dst, const std::vector<T>& v) {
  HS_CUDA(cudaMalloc(dst, std::max<size_t>(v.size(), 1) * sizeof(T)));
  if (!v.empty())
    HS_CUDA(cudaMemcpy(*dst, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice));
}

// Items of the fused CG tail: row j's entry list (N - j column partials,
// then its row segments and split-tile extras) cut into near-equal pieces of
// at most TAIL_ITEM entries; the grid is what fits co-resident.
static void build_tail_plan(hs_matrix* m, SymvPlan* p, const std::vector<int64_t>& row_rseg,
                            const std::vector<int32_t>& row_extra) {
  // opt-in (HS_CG_TAIL=1): measured no faster than finalize + two vector
  // kernels on B200 -- its phase 1 re-reads the same 34 MB of
  // partial slots and the per-CTA round trips, not launches, set the time
  static const bool on = [] {
    const char* e = getenv("HS_CG_TAIL");
    return e && atoi(e) == 1;
  }();
  if (!on) return;
  const int64_t N = (int64_t)m->N, b = (int64_t)m->b;
  int per_sm = 0;
  HS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, cg_tail_kernel, TAIL_THREADS, 0));
  if (per_sm < 1) return;
  std::vector<int4> item;
  std::vector<int2> aux;
  std::vector<int32_t> row_item(N + 1, 0);
  for (int64_t j = 0; j < N; ++j) {
    const int64_t nrs = row_rseg[j + 1] - row_rseg[j];
    const int64_t E = (N - j) + nrs + (row_extra[j + 1] - row_extra[j]);
    const int64_t mj = std::max<int64_t>(1, (E + TAIL_ITEM - 1) / TAIL_ITEM);
    row_item[j] = (int32_t)item.size();
    for (int64_t k = 0; k < mj; ++k) {
      item.push_back(make_int4((int)j, (int)(E * k / mj), (int)(E * (k + 1) / mj),
                               (int)row_rseg[j]));
      aux.push_back(make_int2((int)nrs, (int)row_extra[j]));
    }
  }
  row_item[N] = (int32_t)item.size();
  p->nitems = (int64_t)item.size();
  p->tail_grid = std::min(per_sm, 4) * std::max(1, m->ctx->num_sms);
  upload_vec(&p->item, item);
  upload_vec(&p->item_aux, aux);
  upload_vec(&p->row_item, row_item);
  upload_vec(&p->tail_bar, std::vector<unsigned>(2, 0u));
  HS_CUDA(cudaMalloc(&p->itempart, (size_t)p->nitems * b * sizeof(double)));
  HS_CUDA(cudaMalloc(&p->tail_dot, (size_t)p->tail_grid * sizeof(double)));
  HS_CUDA(cudaMalloc(&p->tail_rr, (size_t)p->tail_grid * sizeof(double)));
}


// Static work plan of the SYMV + finalize pair for one matrix (host side).
void ensure_plan(hs_matrix* m) {
  if (m->plan) return;
  const int64_t b = (int64_t)m->b;
  HS_REQUIRE(m->layout == 0 || m->ctx->world == 1, HS_ERR_CONFIG,
             "CG needs a row-sharded matrix (hs_matrix_create), not a cyclic one");
  HS_REQUIRE(fast_b(m->b) || m->ctx->world == 1, HS_ERR_CONFIG,
             "multi-GPU CG needs block size 64, 128, 256 or 512");
  SymvPlan* p = new SymvPlan;
  if (!fast_b(m->b)) {  // generic kernel needs no plan
    m->plan = p;
    return;
  }
  const int64_t spt = b * b / 4096;
  const int64_t T = m->tile_hi - m->tile_lo;
  const int64_t S = T * spt;
  const int64_t lo = (int64_t)m->row_lo, hi = (int64_t)m->row_hi;
  const int64_t sms = std::max(1, m->ctx->num_sms);
  // Work units, claimed dynamically by the persistent CTAs in this order.
  // Measured per-SM streaming rates differ by up to 20 % on a B200 (44-54
  // GB/s per CTA, fixed by SM position), so a static equal split leaves the
  // fastest CTAs idle for the last ~15 % of the launch. Guided sizes:
  // remaining / (2 * SMs), at least kMinUnit slabs, so the final units are
  // short (a few us) and CTAs finish together. A unit is processed exactly
  // like a static CTA range (its own row / split-tile partial slots), so the
  // sums do not depend on which CTA claims it.
  constexpr int64_t kMinUnit = 8;
  // progressive mode for whole-tile units (b <= 128); HS_CG_PROG=0 keeps the
  // memory-order walk with a finalize after the SYMV
  static const bool prog_on = [] {
    const char* e = getenv("HS_CG_PROG");
    return !(e && atoi(e) == 0);
  }();
  if (spt <= 4 && prog_on && T > 0) {
    // units over the tiles in the order: block row hi-1 (columns 0..hi-1),
    // then hi-2, ..., lo; guided sizes as below, in whole tiles
    const int64_t min_tiles = std::max<int64_t>(1, kMinUnit / spt);
    std::vector<int4> unit_pos;
    std::vector<int32_t> row_seg0(hi, 0), row_nseg(hi, 0);
    int64_t k = hi - 1, j = 0, done_t = 0, nseg = 0;
    while (done_t < T) {
      const int64_t rem = T - done_t;
      const int64_t sz = std::min(rem, std::max(min_tiles, rem / (2 * sms)));
      unit_pos.push_back(make_int4((int)k, (int)j, (int)sz, (int)nseg));
      for (int64_t n = 0; n < sz; ++n) {
        if (n == 0 || j == 0) {  // a new (unit, block row) segment
          if (row_nseg[k] == 0) row_seg0[k] = (int32_t)nseg;
          ++row_nseg[k];
          ++nseg;
        }
        if (j == k) {
          --k;
          j = 0;
        } else {
          ++j;
        }
      }
      done_t += sz;
    }
    p->prog = true;
    p->vgrid = (int)unit_pos.size();
    p->grid = (int)std::max<int64_t>(1, std::min<int64_t>(sms, p->vgrid));
    p->slabs_per_tile = spt;
    p->nrseg = nseg;
    {
      // the heads of the units claimed first (2 tiles, within the block row)
      static const int pf_tiles = [] {
        const char* e = getenv("HS_SYMV_PF_TILES");
        return e ? atoi(e) : 2;
      }();
      std::vector<int64_t> pf;
      for (int64_t u = 0; u < std::min<int64_t>(sms, (int64_t)unit_pos.size()); ++u) {
        const int4 up = unit_pos[u];
        const int64_t nt = std::min<int64_t>({(int64_t)pf_tiles, (int64_t)up.z,
                                              (int64_t)(up.x - up.y + 1)});
        pf.push_back((tri(up.x, up.y) - m->tile_lo) * b * b * 8);
        pf.push_back(std::max<int64_t>(0, nt) * b * b * 8);
      }
      p->pf_units = (int)(pf.size() / 2);
      upload_vec(&p->pf, pf);
    }
    upload_vec(&p->unit_pos, unit_pos);
    upload_vec(&p->row_seg0, row_seg0);
    upload_vec(&p->row_nseg, row_nseg);
    upload_vec(&p->rowdone, std::vector<uint32_t>(2 * hi, 0u));
    upload_vec(&p->unit_ctr, std::vector<uint32_t>(4, 0u));
    // dummies for the memory-order arrays (unused in this mode)
    upload_vec(&p->cta_slab, std::vector<int64_t>(1, 0));
    upload_vec(&p->cta_rseg, std::vector<int64_t>(1, 0));
    HS_CUDA(cudaMalloc(&p->rowpart, std::max<int64_t>(1, nseg) * b * sizeof(double)));
    HS_CUDA(cudaMalloc(&p->colmain, std::max<int64_t>(1, T) * b * sizeof(double)));
    m->plan = p;
    return;
  }
  std::vector<int64_t> cta_slab;
  // slab indices are GLOBAL (the kernel derives global tile / block-row
  // indices from them): this rank's slabs start at tile_lo * spt
  const int64_t s_lo = m->tile_lo * spt;
  {
    int64_t g = 0;
    cta_slab.push_back(s_lo);
    while (g < S) {
      const int64_t rem = S - g;
      int64_t sz = std::min(rem, std::max(kMinUnit, rem / (2 * sms)));
      // b <= 128: whole tiles per unit (the kernel's tile-level loop)
      if (spt <= 4) sz = std::min(rem, (sz + spt - 1) / spt * spt);
      g += sz;
      cta_slab.push_back(s_lo + g);
    }
    if (S == 0) cta_slab.push_back(s_lo);
  }
  const int64_t vgrid = (int64_t)cta_slab.size() - 1;
  const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(sms, vgrid));
  std::vector<int64_t> cta_rseg(vgrid);
  std::vector<int64_t> row_cnt(hi - lo + 1, 0);
  std::vector<std::vector<int32_t>> extras(hi);
  int64_t nr = 0;
  for (int64_t c = 0; c < vgrid; ++c) {
    cta_rseg[c] = nr;
    const int64_t g0 = cta_slab[c], g1 = cta_slab[c + 1];
    if (g0 >= g1) continue;
    const int64_t t0 = g0 / spt, t1 = (g1 - 1) / spt;
    const int64_t i0 = tile_row(t0), i1 = tile_row(t1);
    for (int64_t i = i0; i <= i1; ++i) row_cnt[i - lo]++;
    nr += i1 - i0 + 1;
    if (g0 % spt != 0) extras[t0 - tri(i0, 0)].push_back((int32_t)c);
  }
  std::vector<int64_t> row_rseg(hi - lo + 1, 0);
  for (int64_t i = 0; i < hi - lo; ++i) row_rseg[i + 1] = row_rseg[i] + row_cnt[i];
  std::vector<int32_t> row_extra(hi + 1, 0), extra_cta;
  for (int64_t j = 0; j < hi; ++j) {
    for (int32_t c : extras[j]) extra_cta.push_back(c);
    row_extra[j + 1] = (int32_t)extra_cta.size();
  }
  p->grid = (int)grid;
  p->vgrid = (int)vgrid;
  p->slabs_per_tile = spt;
  p->nrseg = nr;
  upload_vec(&p->cta_slab, cta_slab);
  upload_vec(&p->cta_rseg, cta_rseg);
  upload_vec(&p->row_rseg, row_rseg);
  upload_vec(&p->row_extra, row_extra);
  upload_vec(&p->extra_cta, extra_cta);
  upload_vec(&p->unit_ctr, std::vector<uint32_t>(2, 0u));
  HS_CUDA(cudaMalloc(&p->rowpart, std::max<int64_t>(1, nr) * b * sizeof(double)));
  HS_CUDA(cudaMalloc(&p->colmain, std::max<int64_t>(1, T) * b * sizeof(double)));
  HS_CUDA(cudaMalloc(&p->colextra, std::max<int64_t>(1, vgrid) * b * sizeof(double)));
  if (m->ctx->world == 1 && !m->ctx->distributed()) build_tail_plan(m, p, row_rseg, row_extra);
  m->plan = p;
}


// Progressive-mode outputs of one SYMV launch (the in-kernel finalize)
struct ProgOut {
  double* out = nullptr;
  const double* dot_s = nullptr;
  double* apart = nullptr;
  bool defer = false;
  StepArgs sa{};
  // two-vector mode: out2 = A s2 in the same pass
  const double* s2 = nullptr;
  double* out2 = nullptr;
};

template <int B, int NCW, bool PROG, bool TWO = false>
static void launch_symv_fast(hs_ctx* c, const hs_matrix* m, const double* s,
                             const int32_t* done, const ProgOut* po = nullptr) {
  using Cfg = SymvCfg<B, NCW, PROG, TWO>;
  static std::atomic<uint64_t> attr{0};
  HS_CUDA(smem_attr_once(symv_slab_kernel<B, NCW, PROG, TWO>, Cfg::SMEM, attr));
  SymvPlan* p = m->plan;
  SymvArgs a{};
  a.a = m->d;
  a.s = s;
  a.row_off = m->d_row_off;
  a.tile_lo = m->tile_lo;
  a.cta_slab = p->cta_slab;
  a.cta_rseg = p->cta_rseg;
  a.rowpart = p->rowpart;
  a.colmain = p->colmain;
  a.colextra = p->colextra;
  a.done = done;
  a.unit_ctr = p->unit_ctr;
  a.vgrid = p->vgrid;
  if constexpr (PROG) {
    const int par = (int)(p->launch_seq & 1);
    const int64_t rows = (int64_t)m->row_hi;
    a.prog = 1;
    a.unit_pos = p->unit_pos;
    a.unit_ctr = p->unit_ctr + par;
    a.unit_ctr_next = p->unit_ctr + (par ^ 1);
    a.arrivals = p->unit_ctr + 2 + par;
    a.arrivals_next = p->unit_ctr + 2 + (par ^ 1);
    a.nseg = (uint32_t)p->nrseg;
    a.pf = p->pf;
    a.pf_units = p->pf_units;
    a.rowdone = p->rowdone + par * rows;
    a.rowdone_next = p->rowdone + (par ^ 1) * rows;
    a.row_seg0 = p->row_seg0;
    a.row_nseg = p->row_nseg;
    a.row_lo = (int64_t)m->row_lo;
    a.row_hi = rows;
    a.out = po->out;
    a.dot_s = po->dot_s;
    a.apart = po->apart;
    a.defer = po->defer ? 1 : 0;
    a.sa = po->sa;
    ++p->launch_seq;
  }
#ifdef HS_SYMV_TIMING
  static unsigned seq = 0;
  a.ts_seq = seq++;
#endif
  if constexpr (TWO) {
    a.s2 = po->s2;
    a.out2 = po->out2;
    a.rowpart2 = p->rowpart2;
    a.colmain2 = p->colmain2;
  }
  HS_CUDA(launch_pdl(symv_slab_kernel<B, NCW, PROG, TWO>, dim3(p->grid), dim3(Cfg::THREADS),
                     Cfg::SMEM, c->stream, a));
  HS_CUDA(cudaGetLastError());
  launch_count(c);
}

static void ensure_dpart(hs_ctx* c, size_t count) {
  if (c->dpart_cap >= count) return;
  cudaFree(c->d_dpart);
  HS_CUDA(cudaMalloc(&c->d_dpart, count * sizeof(double)));
  c->dpart_cap = count;
}

// SYMV over the rank's tiles into `out` (padded full layout). With fuse_dot,
// also dot(s, out) in the finalize and the ALPHA step (single rank), or the
// rank's s^T t partial into the dot slots (multi-rank).
static void symv_to(hs_ctx* c, const hs_matrix* m, const double* s, double* out,
                    bool fuse_dot, const StepArgs* sa, const int32_t* done,
                    double* defer_alpha = nullptr, bool finalize = true) {
  const int b = (int)m->b;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  const bool prof = c->prof && (c->prof_counter++ % c->prof_every == 0);
  if (prof) {
    HS_CUDA(cudaEventCreate(&e0));
    HS_CUDA(cudaEventCreate(&e1));
    HS_CUDA(cudaEventRecord(e0, c->stream));
  }
  if (!fast_b(m->b)) {
    const int64_t pn = (int64_t)m->N * b;
    const int64_t threads = pn * 32;
    HS_CUDA(launch_pdl(symv_generic_kernel, dim3((unsigned)ceil_div(threads, 256)), dim3(256),
                       0, c->stream, (const double*)m->d, pn, b, s, out, done));
    HS_CUDA(cudaGetLastError());
    launch_count(c);
    if (prof) {
      HS_CUDA(cudaEventRecord(e1, c->stream));
      c->prof_events.push_back(e0);
      c->prof_events.push_back(e1);
    }
    if (fuse_dot) {
      VecArgs va{};
      va.len = pn;
      va.s = const_cast<double*>(s);
      va.t = out;
      va.dpart = c->d_dpart;
      va.sa = *sa;
      va.done = done;
      va.mode = V_DOT_ST;
      HS_CUDA(launch_pdl(vec_kernel, dim3(VGRID), dim3(VBLOCK), 0, c->stream, va));
      launch_count(c);
    }
    return;
  }
  SymvPlan* p = m->plan;
  if (p->prog) {
    // one launch: the SYMV's finalize warps form t (and s . t) as the
    // block rows complete
    ProgOut po;
    po.out = out;
    po.dot_s = fuse_dot ? s : nullptr;
    po.apart = defer_alpha ? defer_alpha : c->d_dpart + VGRID + 8;  // per-block-row s . t
    po.defer = defer_alpha != nullptr;
    if (sa) po.sa = *sa;
    if (b == 64) launch_symv_fast<64, 8, true>(c, m, s, done, &po);
    else launch_symv_fast<128, 8, true>(c, m, s, done, &po);
    if (prof) {
      HS_CUDA(cudaEventRecord(e1, c->stream));
      c->prof_events.push_back(e0);
      c->prof_events.push_back(e1);
    }
    return;
  }
  switch (b) {
    case 64: launch_symv_fast<64, 8, false>(c, m, s, done); break;
    case 128: launch_symv_fast<128, 8, false>(c, m, s, done); break;
    case 256: launch_symv_fast<256, 8, false>(c, m, s, done); break;
    case 512: launch_symv_fast<512, 8, false>(c, m, s, done); break;
  }
  if (prof) {
    HS_CUDA(cudaEventRecord(e1, c->stream));
    c->prof_events.push_back(e0);
    c->prof_events.push_back(e1);
  }
  if (!finalize) return;  // the fused CG tail consumes the partial slots
  FinalizeArgs fa{};
  fa.row_rseg = p->row_rseg;
  fa.row_extra = p->row_extra;
  fa.extra_cta = p->extra_cta;
  fa.rowpart = p->rowpart;
  fa.colmain = p->colmain;
  fa.colextra = p->colextra;
  fa.unit_ctr = p->unit_ctr;
#ifdef HS_SYMV_TIMING
  static unsigned fseq = 0;
  fa.ts_seq = fseq++;
#endif
  fa.row_off = m->d_row_off;
  fa.row_lo = (int64_t)m->row_lo;
  fa.row_hi = (int64_t)m->row_hi;
  fa.tile_lo = m->tile_lo;
  fa.b = b;
  fa.out = out;
  fa.s = fuse_dot ? s : nullptr;
  fa.dpart = c->d_dpart;
  fa.apart = fuse_dot ? defer_alpha : nullptr;
  fa.step = STEP_ALPHA;
  if (sa) fa.sa = *sa;
  fa.done = done;
  {
    // slabs of every unit's head prefetched into L2 for the next SYMV
    // (HS_SYMV_PF_SLABS overrides, 0 disables)
    static const int pf = [] {
      const char* e = getenv("HS_SYMV_PF_SLABS");
      return e ? atoi(e) : 8;
    }();
    fa.pf_base = reinterpret_cast<const unsigned char*>(m->d);
    fa.pf_slab = p->cta_slab;
    fa.pf_slab_lo = m->tile_lo * p->slabs_per_tile;
    fa.pf_units = std::min(p->grid, p->vgrid);
    fa.pf_slabs = pf;
  }
  HS_CUDA(launch_pdl(finalize_kernel, dim3((unsigned)m->row_hi, (unsigned)(b / FIN_COLS)),
                     dim3(FIN_THREADS), 0, c->stream, fa));
  HS_CUDA(cudaGetLastError());
  launch_count(c);
}

// Two matvecs in one pass over A (progressive mode, b <= 128): out = A s
// (with s . out deferred into apart, as the plain CG iteration) and
// out2 = A s2. The CG recompute iteration uses it for A s and A x.
static void symv2_to(hs_ctx* c, const hs_matrix* m, const double* s, const double* s2,
                     double* out, double* out2, const StepArgs& sa, const int32_t* done,
                     double* apart, bool defer) {
  SymvPlan* p = m->plan;
  const int64_t b = (int64_t)m->b;
  if (!p->colmain2) {
    HS_CUDA(cudaStreamSynchronize(c->stream));
    const int64_t T = m->tile_hi - m->tile_lo;
    HS_CUDA(cudaMalloc(&p->rowpart2, std::max<int64_t>(1, p->nrseg) * b * sizeof(double)));
    HS_CUDA(cudaMalloc(&p->colmain2, std::max<int64_t>(1, T) * b * sizeof(double)));
  }
  ProgOut po;
  po.out = out;
  po.dot_s = s;
  po.apart = apart;
  po.defer = defer;
  po.sa = sa;
  po.s2 = s2;
  po.out2 = out2;
  if (b == 64) launch_symv_fast<64, 8, true, true>(c, m, s, done, &po);
  else launch_symv_fast<128, 8, true, true>(c, m, s, done, &po);
}

// The fused tail after a plain single-rank SYMV: cooperative launch (the
// grid barriers need every CTA resident), programmatic serialization when
// the driver accepts both attributes together.
static void launch_tail(hs_ctx* c, const hs_matrix* m, double* x, double* r, double* s,
                        const StepArgs& sa, const int32_t* done) {
  SymvPlan* p = m->plan;
  TailArgs ta{};
  ta.rowpart = p->rowpart;
  ta.colmain = p->colmain;
  ta.colextra = p->colextra;
  ta.extra_cta = p->extra_cta;
  ta.unit_ctr = p->unit_ctr;
  ta.N = (int64_t)m->N;
  ta.b = (int)m->b;
  ta.nch = (int)(m->b / 32);
  ta.lgb = 0;
  while ((1 << ta.lgb) < ta.b) ++ta.lgb;
  ta.item = p->item;
  ta.item_aux = p->item_aux;
  ta.row_item = p->row_item;
  ta.nitems = p->nitems;
  ta.itempart = p->itempart;
  ta.dotpart = p->tail_dot;
  ta.rrpart = p->tail_rr;
  ta.bar = p->tail_bar;
  ta.len = (int64_t)(m->N * m->b);
  ta.x = x;
  ta.r = r;
  ta.s = s;
  ta.sa = sa;
  ta.done = done;
#ifdef HS_SYMV_TIMING
  static unsigned tseq = 0;
  ta.ts_seq = tseq++;
#endif
  static const int pf = [] {
    const char* e = getenv("HS_SYMV_PF_SLABS");
    return e ? atoi(e) : 8;
  }();
  ta.pf_base = reinterpret_cast<const unsigned char*>(m->d);
  ta.pf_slab = p->cta_slab;
  ta.pf_slab_lo = m->tile_lo * p->slabs_per_tile;
  ta.pf_units = std::min(p->grid, p->vgrid);
  ta.pf_slabs = pf;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)p->tail_grid);
  cfg.blockDim = dim3(TAIL_THREADS);
  cfg.stream = c->stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  // 0 unknown, 1 cooperative + PDL accepted, 2 cooperative only;
  // HS_CG_TAIL_LAUNCH: 3 = plain PDL launch (diagnostics: no co-residency
  // guarantee), 2 = cooperative without PDL
  static std::atomic<int> mode{[] {
    const char* e = getenv("HS_CG_TAIL_LAUNCH");
    return e ? atoi(e) : 0;
  }()};
  int md = mode.load();
  if (md == 3) {
    cfg.attrs = attr + 1;
    cfg.numAttrs = 1;
    HS_CUDA(cudaLaunchKernelEx(&cfg, cg_tail_kernel, ta));
    launch_count(c);
    return;
  }
  cudaError_t e = cudaSuccess;
  if (md != 2) {
    cfg.numAttrs = 2;
    e = cudaLaunchKernelEx(&cfg, cg_tail_kernel, ta);
    if (e == cudaSuccess) {
      mode.store(1);
    } else if (md == 0) {
      cudaGetLastError();
      mode.store(2);
      md = 2;
    }
  }
  if (md == 2) {
    cfg.numAttrs = 1;
    e = cudaLaunchKernelEx(&cfg, cg_tail_kernel, ta);
  }
  HS_CUDA(e);
  launch_count(c);
}

void symv_local(hs_ctx* c, const hs_matrix* m, const double* x, double* y) {
  ensure_plan(const_cast<hs_matrix*>(m));
  symv_to(c, m, x, y, false, nullptr, nullptr);
}

static void launch_vec(hs_ctx* c, VecArgs va) {
  HS_CUDA(launch_pdl(vec_kernel, dim3(VGRID), dim3(VBLOCK), 0, c->stream, va));
  HS_CUDA(cudaGetLastError());
  launch_count(c);
}

// ---------------------------------------------------------------------------
// CG driver

// CG vectors, carved from the context's persistent workspace (grown when a
// call needs more, never freed per call)
struct CgBuffers {
  double* s_full = nullptr;  // padded full layout (vec_len)
  double* x_full = nullptr;  // padded full layout (recompute / result)
  double* t = nullptr;       // partial (vec_len) or local result (world 1)
  double* t2 = nullptr;      // A x_old of the two-vector recompute (partial if multi-rank)
  double* t2_loc = nullptr;  // its reduced own rows (multi-rank)
  double* r_full = nullptr;  // multi-rank: all-gathered r chunks (+ slots)
  double* t_loc = nullptr;   // reduced own rows (multi-rank)
  double* r = nullptr;       // local chunk
  double* rhs = nullptr;     // local chunk
  double* trace = nullptr;   // device trace
  Dd* slots = nullptr;       // [world] gathered partials
};

static void carve_cg_buffers(hs_ctx* c, CgBuffers& B, int64_t full, int64_t chunk, int world,
                             size_t trace_n, bool dp) {
  struct Req {
    void** p;
    size_t bytes;
  };
  const Req req[] = {
      {(void**)&B.s_full, full * sizeof(double)},
      {(void**)&B.x_full, full * sizeof(double)},
      {(void**)&B.t, full * sizeof(double)},
      {(void**)&B.t2, full * sizeof(double)},
      {(void**)&B.r, chunk * sizeof(double)},
      {(void**)&B.r_full, dp ? full * sizeof(double) : 0},
      {(void**)&B.rhs, chunk * sizeof(double)},
      {(void**)&B.slots, std::max(world, 1) * sizeof(Dd)},
      {(void**)&B.t_loc, dp ? chunk * sizeof(double) : 0},
      {(void**)&B.t2_loc, dp ? chunk * sizeof(double) : 0},
      {(void**)&B.trace, 3 * trace_n * sizeof(double)},
  };
  auto up = [](size_t x) { return (x + 255) & ~(size_t)255; };
  size_t total = 0;
  for (const Req& q : req) total += up(q.bytes);
  if (total > c->cg_ws_bytes) {
    HS_CUDA(cudaStreamSynchronize(c->stream));
    cudaFree(c->cg_ws);
    c->cg_ws = nullptr;
    c->cg_ws_bytes = 0;
    HS_CUDA(cudaMalloc(&c->cg_ws, total));
    c->cg_ws_bytes = total;
  }
  char* base = static_cast<char*>(c->cg_ws);
  for (const Req& q : req) {
    *q.p = q.bytes ? base : nullptr;
    base += up(q.bytes);
  }
}

static double ms_since(std::chrono::steady_clock::time_point t0) {
  return std::chrono::duration<double, std::milli>(
             std::chrono::steady_clock::now() - t0)
      .count();
}

// d_rhs / d_x: full standard-layout vectors (N*b) on this rank's GPU.
static void cg_run(hs_ctx* c, const hs_matrix* m, const double* d_rhs,
                   const hs_cg_params* prm, double* d_x, hs_cg_stats* st,
                   double* h_trace) {
  HS_REQUIRE(prm->eps > 0.0, HS_ERR_CONFIG, "eps must be positive");
  // HS_CG_HOST_TIMING=1: host-side phase times of this call on stderr
  static const bool host_timing = getenv("HS_CG_HOST_TIMING") != nullptr;
  const auto ht0 = std::chrono::steady_clock::now();
  auto ht = [&](const char* what) {
    if (host_timing) {
      const auto now = std::chrono::steady_clock::now();
      fprintf(stderr, "cg_run %-10s %9.3f ms (monotonic %.3f ms)\n", what,
              std::chrono::duration<double, std::milli>(now - ht0).count(),
              std::chrono::duration<double, std::milli>(now.time_since_epoch()).count());
    }
  };
  ht("enter");
  ensure_plan(const_cast<hs_matrix*>(m));
  const int world = c->world, rank = c->rank;
  // distributed protocol whenever there is a communicator (also world == 1,
  // which runs the NCCL path on one GPU)
  const bool dp = c->distributed();
  const int64_t b = (int64_t)m->b;
  const int64_t N = (int64_t)m->N;
  const int64_t chunk = m->vec_len / world;  // doubles per rank chunk
  const int64_t full = m->vec_len;
  const int64_t rows_len = m->slot_off;      // row part of a chunk
  const int64_t lo = (int64_t)m->row_lo, hi = (int64_t)m->row_hi;
  const int64_t own = (hi - lo) * b;  // valid doubles in the chunk
  const size_t trace_n = prm->record_trace ? (size_t)prm->max_iters : 0;
  const bool rec_on = prm->recompute_interval > 0;

  // finalize / vector partials, and (after VGRID + 8) the deferred-alpha
  // partials of the single-rank iteration
  ensure_dpart(c, std::max<int64_t>({N * b / FIN_COLS + VGRID + 8, N + 1, VGRID}));
  double* apart = c->d_dpart + VGRID + 8;
  // deferred-alpha partials: one per finalize CTA (N * b / 32), or one per
  // block row in the progressive mode
  const int acount = m->plan->prog ? (int)m->row_hi : (int)(N * b / FIN_COLS);
  CgBuffers B;
  // single rank + fast SYMV: the direction update rides inside the SYMV
  // (double-buffered s); otherwise a separate vector kernel does it
  carve_cg_buffers(c, B, full, chunk, world, trace_n, dp);
  HS_CUDA(cudaMemsetAsync(B.t, 0, full * sizeof(double), c->stream));
  // (rows a rank's SYMV never writes -- padding, rows past its last block
  // row -- stay zero for the reduce-scatters)
  HS_CUDA(cudaMemsetAsync(B.t2, 0, full * sizeof(double), c->stream));
  HS_CUDA(cudaMemsetAsync(B.r, 0, chunk * sizeof(double), c->stream));
  HS_CUDA(cudaMemsetAsync(B.rhs, 0, chunk * sizeof(double), c->stream));
  HS_CUDA(cudaMemsetAsync(B.x_full, 0, full * sizeof(double), c->stream));
  HS_CUDA(cudaMemsetAsync(c->d_scalars, 0, sizeof(CgScalars), c->stream));
  // own rows of rhs into the local chunk (standard layout -> chunk)
  HS_CUDA(cudaMemcpyAsync(B.rhs, d_rhs + lo * b, own * sizeof(double),
                          cudaMemcpyDeviceToDevice, c->stream));

  double* s_loc = B.s_full + (int64_t)rank * chunk;
  double* x_loc = B.x_full + (int64_t)rank * chunk;
  double* t_own = dp ? B.t_loc : B.t;
  const int32_t* done = &c->d_scalars->done;

  // sa.world == 1: the last CTA applies the scalar step itself; otherwise it
  // publishes its (hi, lo) partial for the all-gather + rank-ordered combine
  StepArgs sa{c->d_scalars, B.trace, prm->eps, B.slots, dp ? 0 : 1};

  auto dot_finish = [&](int step) {
    if (!dp) return;
    // all-gather the (hi, lo) partials in place, combine in rank order
    comm_allgather(c, reinterpret_cast<double*>(B.slots) + 2 * rank,
                   reinterpret_cast<double*>(B.slots), 2, LK_SCALAR);
    combine_kernel<<<1, 1, 0, c->stream>>>(B.slots, 1, world, step, sa, nullptr,
                                           done);
    HS_CUDA(cudaGetLastError());
    launch_count(c);
  };
  // In the multi-rank kernels the local partial is written to slots[0];
  // relocate it into this rank's slot before the in-place all-gather.
  StepArgs sa_local = sa;
  sa_local.dd_slots = B.slots + rank;
  // per-iteration dots ride in the chunk slots (see the loop)
  StepArgs sa_alpha = sa, sa_beta = sa;
  sa_alpha.dd_slots = reinterpret_cast<Dd*>(B.t + rows_len) + rank;
  sa_alpha.slot_stride = chunk / 2;
  sa_alpha.slot_count = world;
  sa_beta.dd_slots = reinterpret_cast<Dd*>(B.r + rows_len) + rank;

  static const bool recomp2_env = [] {
    const char* e = getenv("HS_CG_RECOMP2");
    return !(e && atoi(e) == 0);
  }();
  const bool two_pass_ok = recomp2_env && m->plan->prog;
  VecArgs v{};
  v.len = rows_len;  // the chunk's rows (its slot region is not vector data)
  v.x = x_loc;
  v.r = B.r;
  v.s = s_loc;
  v.t = t_own;
  v.rhs = B.rhs;
  v.dpart = c->d_dpart;
  v.sa = dp ? sa_local : sa;
  v.done = done;

  // x0 = 0, r = s = rhs, u0 = rhs^T rhs (cg_solver.cpp:243-249)
  v.mode = V_INIT;
  launch_vec(c, v);
  c->step = -1;  // ledger: setup
  dot_finish(STEP_INIT);
  if (dp) {
    comm_allgather(c, s_loc, B.s_full, (size_t)chunk, LK_SUBVECTOR);
    v.sa = sa_beta;  // r^T r partials ride in the r all-gather
  }

  // Convergence is decided on the device (done flag); the host polls a
  // pinned copy of the scalars one chunk behind, so the GPU queue never
  // drains while the host checks.
  // poll points every 4 iterations at first (a converging solve stops at
  // most two chunks late), then every 16 / 32: long runs keep 20-40 ms of
  // work queued, so a host thread delayed by the OS does not drain the GPU
  uint64_t next_poll = 4, polls = 0;
  auto poll_gap = [](uint64_t it) -> uint64_t { return it < 64 ? 4 : it < 256 ? 16 : 32; };
  CgScalars* pin = reinterpret_cast<CgScalars*>(c->h_pinned);
  struct PollEvents {  // destroyed on every exit path, including throws
    cudaEvent_t e[2] = {nullptr, nullptr};
    ~PollEvents() {
      for (cudaEvent_t x : e)
        if (x) cudaEventDestroy(x);
    }
  } pe;
  cudaEvent_t* ev = pe.e;
  HS_CUDA(cudaEventCreateWithFlags(&ev[0], cudaEventDisableTiming));
  HS_CUDA(cudaEventCreateWithFlags(&ev[1], cudaEventDisableTiming));
  int pending = -1;
  CgScalars h{};
  ht("setup");
  for (uint64_t it = 1; it <= prm->max_iters; ++it) {
    c->step = (int64_t)it;
    const bool recompute = rec_on && (it % prm->recompute_interval == 0);
    // single rank, fast b, plain iteration: alpha is reduced by the update
    // kernel itself from the finalize's partials (no last-CTA tail)
    const bool defer = !dp && fast_b(m->b) && !recompute;
    if (defer && m->plan->tail_grid > 0) {
      // lines 4-11 in two launches: the SYMV, then the fused tail (t,
      // alpha, x, r, r^T r, beta, s)
      symv_to(c, m, B.s_full, B.t, false, nullptr, done, nullptr, false);
      launch_tail(c, m, x_loc, B.r, s_loc, sa, done);
      goto poll;
    }
    // recompute iteration, single rank, progressive SYMV: A s and A x_old in
    // one pass over A, then x += alpha s and r = rhs - (A x_old + alpha A s)
    // (= rhs - A x_new, cg_solver.cpp:277-298) in one vector kernel
    // (HS_CG_RECOMP2=0: two passes as below)
    if (recompute && two_pass_ok && !dp) {
      symv2_to(c, m, B.s_full, B.x_full, B.t, B.t2, sa, done, apart, true);
      VecArgs vr = v;
      vr.mode = V_RECOMP;
      vr.apart = apart;
      vr.acount = acount;
      vr.t2 = B.t2;
      launch_vec(c, vr);
      v.mode = V_SDIR;
      launch_vec(c, v);
      goto poll;
    }
    if (recompute && two_pass_ok && dp) {
      // the same collectives as the two-pass recompute (one all-gather of
      // x, two reduce-scatters), one pass over the local tiles: x_old to
      // every rank first, then A s and A x_old together
      comm_allgather(c, x_loc, B.x_full, (size_t)chunk, LK_SUBVECTOR);
      symv2_to(c, m, B.s_full, B.x_full, B.t, B.t2, sa_alpha, done, apart, false);
      comm_reduce_scatter(c, B.t, B.t_loc, (size_t)chunk, LK_SUBVECTOR);
      combine_kernel<<<1, 1, 0, c->stream>>>(
          reinterpret_cast<const Dd*>(B.t_loc + rows_len), 1, world, STEP_ALPHA, sa,
          nullptr, done);
      HS_CUDA(cudaGetLastError());
      launch_count(c);
      comm_reduce_scatter(c, B.t2, B.t2_loc, (size_t)chunk, LK_SUBVECTOR);
      VecArgs vr = v;
      vr.mode = V_RECOMP;
      vr.t2 = B.t2_loc;
      launch_vec(c, vr);
      goto dp_tail;
    }
    // lines 4-5: t = A s, alpha = u / s^T t (the dot fused into the finalize)
    if (!dp) {
      symv_to(c, m, B.s_full, B.t, true, &sa, done, defer ? apart : nullptr);
    } else {
      // s^T t = sum over ranks of s^T (this rank's partial t): the finalize
      // forms it on the full-length partial and writes the (hi, lo) into
      // slot `rank` of every rank chunk of t (other slots stay 0), so the
      // reduce-scatter that sums t also hands every rank all W partials,
      // exactly; combined in rank order -> alpha, identical everywhere
      symv_to(c, m, B.s_full, B.t, true, &sa_alpha, done);
      comm_reduce_scatter(c, B.t, B.t_loc, (size_t)chunk, LK_SUBVECTOR);
      combine_kernel<<<1, 1, 0, c->stream>>>(
          reinterpret_cast<const Dd*>(B.t_loc + rows_len), 1, world, STEP_ALPHA, sa,
          nullptr, done);
      HS_CUDA(cudaGetLastError());
      launch_count(c);
    }
    if (recompute) {
      // x += alpha s; r = rhs - A x (cg_solver.cpp:277-298)
      v.mode = V_AXPY_X;
      launch_vec(c, v);
      if (dp) comm_allgather(c, x_loc, B.x_full, (size_t)chunk, LK_SUBVECTOR);
      symv_to(c, m, B.x_full, B.t, false, nullptr, done);
      if (dp) comm_reduce_scatter(c, B.t, B.t_loc, (size_t)chunk, LK_SUBVECTOR);
      v.mode = V_RESIDUAL;
      launch_vec(c, v);
    } else {
      VecArgs vu = v;
      vu.mode = V_UPDATE;  // lines 6-7 + u = r^T r + beta
      if (defer) {
        vu.apart = apart;
        vu.acount = acount;
      }
      launch_vec(c, vu);
    }
  dp_tail:
    if (!dp) {
      // line 11 as its own small kernel: forming s = r + beta s inside the
      // next SYMV (one more staged segment per slab) measured 4 % slower per
      // iteration under the board's power cap
      v.mode = V_SDIR;
      launch_vec(c, v);
    } else {
      // r chunks (+ each rank's r^T r partial in its slot) to every rank;
      // beta from the slots in rank order; s = r + beta s on the full
      // vector by every rank (the arithmetic of the local update + an
      // all-gather of s, without that second collective)
      comm_allgather(c, B.r, B.r_full, (size_t)chunk, LK_SUBVECTOR);
      combine_kernel<<<1, 1, 0, c->stream>>>(
          reinterpret_cast<const Dd*>(B.r_full + rows_len), (chunk + 2) / 2, world,
          STEP_BETA, sa, nullptr, done);
      HS_CUDA(cudaGetLastError());
      launch_count(c);
      VecArgs vs = v;
      vs.len = full;
      vs.r = B.r_full;
      vs.s = B.s_full;
      vs.mode = V_SDIR;
      launch_vec(c, vs);
    }
  poll:
    if (it == next_poll) {
      next_poll += poll_gap(it);
      const int slot = (int)(polls++ & 1);
      HS_CUDA(cudaMemcpyAsync(pin + slot, c->d_scalars, sizeof(CgScalars),
                              cudaMemcpyDeviceToHost, c->stream));
      HS_CUDA(cudaEventRecord(ev[slot], c->stream));
      if (pending >= 0) {
        HS_CUDA(cudaEventSynchronize(ev[pending]));
        if (pin[pending].done) break;
      }
      pending = slot;
    }
  }
  ht("loop");
  HS_CUDA(cudaMemcpyAsync(&h, c->d_scalars, sizeof(CgScalars),
                          cudaMemcpyDeviceToHost, c->stream));
  HS_CUDA(cudaStreamSynchronize(c->stream));
  ht("drained");
  // recomputation count is a pure function of the iteration count
  st->iterations = (uint64_t)h.iter;
  st->recomputations = rec_on ? (uint64_t)h.iter / prm->recompute_interval : 0;
  if (h.status == HS_ERR_NUMERICAL) {
    // an error inside iteration k: iterations completed = k - 1
    st->error_iteration = h.err_iter;
    st->u0 = h.u0;
    throw Failure{HS_ERR_NUMERICAL,
                  h.err_iter == 0 ? std::string("initial residual is not finite")
                                  : "non-finite scalar at iteration " +
                                        std::to_string(h.err_iter),
                  h.err_iter, -1};
  }
  st->converged = h.u <= h.limit ? 1 : 0;
  st->u0 = h.u0;
  st->error_iteration = -1;
  if (trace_n && h_trace && h.iter > 0)
    HS_CUDA(cudaMemcpy(h_trace, B.trace, 3 * (size_t)h.iter * sizeof(double),
                       cudaMemcpyDeviceToHost));

  // result: full x in the standard layout
  c->step = -1;
  if (dp) comm_allgather(c, x_loc, B.x_full, (size_t)chunk, LK_RESULT);
  for (int g = 0; g < world; ++g) {
    const int64_t glo = m->bounds[g], ghi = m->bounds[g + 1];
    if (ghi > glo)
      HS_CUDA(cudaMemcpyAsync(d_x + glo * b, B.x_full + (int64_t)g * chunk,
                              (ghi - glo) * b * sizeof(double),
                              cudaMemcpyDeviceToDevice, c->stream));
  }
  // the solve ends here; the exit diagnostic below is untimed, as in the
  // reference (cg_solver.cpp:354-365)
  HS_CUDA(cudaStreamSynchronize(c->stream));
  st->compute_ms = ms_since(ht0);
  // exit diagnostic: ||rhs - A x|| (cg_solver.cpp:360-365)
  symv_to(c, m, B.x_full, B.t, false, nullptr, nullptr);
  if (dp) comm_reduce_scatter(c, B.t, B.t_loc, (size_t)chunk, LK_SUBVECTOR);
  VecArgs vr = v;
  vr.mode = V_RESNORM;
  vr.done = nullptr;
  if (dp) vr.sa = sa_local;
  launch_vec(c, vr);
  double res2;
  if (dp) {
    comm_allgather(c, reinterpret_cast<double*>(B.slots) + 2 * rank,
                   reinterpret_cast<double*>(B.slots), 2, LK_SCALAR);
    combine_kernel<<<1, 1, 0, c->stream>>>(B.slots, 1, world, STEP_NONE, sa,
                                           c->d_dpart + N, nullptr);
    HS_CUDA(cudaGetLastError());
    launch_count(c);
    HS_CUDA(cudaMemcpyAsync(&res2, c->d_dpart + N, sizeof(double),
                            cudaMemcpyDeviceToHost, c->stream));
  } else {
    // single rank: the epilogue left the DD in dpart via STEP_NONE; redo the
    // fixed-order combine on the host from the per-CTA partials
    std::vector<double> parts(VGRID);
    HS_CUDA(cudaMemcpyAsync(parts.data(), c->d_dpart, VGRID * sizeof(double),
                            cudaMemcpyDeviceToHost, c->stream));
    HS_CUDA(cudaStreamSynchronize(c->stream));
    Dd acc{0.0, 0.0};
    for (double p : parts) acc = dd_add(acc, p);
    res2 = dd_value(acc);
  }
  HS_CUDA(cudaStreamSynchronize(c->stream));
  st->true_residual = sqrt(res2);
  ht("exit");
}

}  // namespace hs

using namespace hs;

#define HS_API_BEGIN \
  clear_error();     \
  try {
#define HS_API_END                                                         \
  return HS_OK;                                                            \
  }                                                                        \
  catch (const Failure& f) {                                               \
    set_error(f.status, f.msg, f.a, f.b);                                  \
    return f.status;                                                       \
  }                                                                        \
  catch (const std::exception& e) {                                        \
    set_error(HS_ERR_CUDA, e.what());                                      \
    return HS_ERR_CUDA;                                                    \
  }

extern "C" {

hs_status hs_symv(hs_ctx* c, const hs_matrix* m, const double* d_x,
                  double* d_y) {
  HS_API_BEGIN
  HS_REQUIRE(c && m && d_x && d_y, HS_ERR_CONFIG, "null pointer");
  HS_REQUIRE(c->world == 1, HS_ERR_CONFIG,
             "hs_symv is single-rank; use hs_cg_solve for sharded matrices");
  HS_CUDA(cudaSetDevice(c->device));
  symv_local(c, m, d_x, d_y);
  HS_CUDA(cudaStreamSynchronize(c->stream));
  HS_API_END
}

// t (full length) = this rank's share of A x over a block-cyclic matrix:
// block row i (blockIdx.y), 32 rows (blockIdx.x), summed over the owned
// tiles (i, j <= i) as rows and (j > i, i) transposed; diagonal tiles use
// their lower triangle only, like the SYMV. Fixed order, no atomics.
__global__ void __launch_bounds__(256)
    cyclic_partial_symv_kernel(const double* A, const int64_t* lpos, const double* x,
                               double* t, int b, int64_t N) {
  const int64_t i = blockIdx.y;
  const int o0 = blockIdx.x * 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t bb = (int64_t)b * b;
  double rowacc[4] = {0.0, 0.0, 0.0, 0.0};  // rows o0 + warp + 8q (lanes over cols)
  double colacc = 0.0;                      // row o0 + lane (warps over tile rows)
  for (int64_t j = 0; j < N; ++j) {
    const double* xj = x + j * b;
    if (j <= i) {
      const int64_t slot = lpos[i * (i + 1) / 2 + j];
      if (slot >= 0) {
        const double* T = A + slot * bb;
        for (int q = 0; q < 4; ++q) {
          const int r = o0 + warp + 8 * q;
          if (r >= b) break;
          const int cend = j == i ? r + 1 : b;
          for (int cc = lane; cc < cend; cc += 32) rowacc[q] = fma(T[(int64_t)r * b + cc], xj[cc], rowacc[q]);
        }
        if (j == i && o0 + lane < b)  // strictly upper part of the diagonal tile
          for (int cc = o0 + lane + 1 + warp; cc < b; cc += 8)
            colacc = fma(T[(int64_t)cc * b + o0 + lane], xj[cc], colacc);
      }
    } else {
      const int64_t slot = lpos[j * (j + 1) / 2 + i];
      if (slot >= 0 && o0 + lane < b) {
        const double* T = A + slot * bb;
        for (int cc = warp; cc < b; cc += 8)
          colacc = fma(T[(int64_t)cc * b + o0 + lane], xj[cc], colacc);
      }
    }
  }
  __shared__ double rows[32], cols[8][33];
  for (int q = 0; q < 4; ++q) {
    double a = rowacc[q];
    for (int off = 16; off; off >>= 1) a += __shfl_xor_sync(0xffffffffu, a, off);
    if (lane == 0) rows[warp + 8 * q] = a;
  }
  cols[warp][lane] = colacc;
  __syncthreads();
  if (warp == 0 && o0 + lane < b) {
    double v = rows[lane];
    for (int w = 0; w < 8; ++w) v += cols[w][lane];
    t[i * b + o0 + lane] = v;
  }
}

// t = sum over ranks of the gathered partials, rank order
__global__ void rank_sum_kernel(const double* G, double* t, int64_t len, int world) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < len;
       k += (int64_t)gridDim.x * blockDim.x) {
    double v = 0.0;
    for (int r = 0; r < world; ++r) v += G[r * len + k];
    t[k] = v;
  }
}

hs_status hs_true_residual(hs_ctx* c, const hs_matrix* m, const double* d_x,
                           const double* d_rhs, double* out) {
  HS_API_BEGIN
  HS_REQUIRE(c && m && d_x && d_rhs && out, HS_ERR_CONFIG, "null pointer");
  HS_REQUIRE(c->world == 1 || m->layout == 1, HS_ERR_CONFIG,
             "multi-rank hs_true_residual needs a block-cyclic matrix (full-length x)");
  HS_CUDA(cudaSetDevice(c->device));
  const int64_t pn = (int64_t)m->N * (int64_t)m->b;
  // scratch from the context's persistent workspace 0
  const size_t sz[2] = {(size_t)pn * sizeof(double),
                        c->world > 1 ? (size_t)pn * c->world * sizeof(double) : 0};
  void* ws[2];
  ctx_workspace(c, 0, sz, 2, ws);
  double* t = static_cast<double*>(ws[0]);
  double* gath = static_cast<double*>(ws[1]);
  {
    if (c->world > 1) {
      // every rank: its owned tiles' share of A x; all-gather; rank-order sum
      const int b = (int)m->b;
      cyclic_partial_symv_kernel<<<dim3((b + 31) / 32, (unsigned)m->N), 256, 0, c->stream>>>(
          m->d, m->d_lpos, d_x, t, b, (int64_t)m->N);
      HS_CUDA(cudaGetLastError());
      launch_count(c);
      c->step = -1;
      comm_allgather(c, t, gath, (size_t)pn, LK_RESULT);
      rank_sum_kernel<<<592, 256, 0, c->stream>>>(gath, t, pn, c->world);
      HS_CUDA(cudaGetLastError());
      launch_count(c);
    } else {
      symv_local(c, m, d_x, t);
    }
    ensure_dpart(c, std::max<int64_t>({(int64_t)(m->N * m->b) / FIN_COLS + 1,
                                       (int64_t)m->N + 1, VGRID}));
    HS_CUDA(cudaMemsetAsync(c->d_scalars, 0, sizeof(CgScalars), c->stream));
    VecArgs v{};
    v.len = pn;
    v.t = t;
    v.rhs = d_rhs;
    v.dpart = c->d_dpart;
    v.sa = StepArgs{c->d_scalars, nullptr, 1.0, nullptr, 1};
    v.mode = V_RESNORM;
    launch_vec(c, v);
    std::vector<double> parts(VGRID);
    HS_CUDA(cudaMemcpyAsync(parts.data(), c->d_dpart, VGRID * sizeof(double),
                            cudaMemcpyDeviceToHost, c->stream));
    HS_CUDA(cudaStreamSynchronize(c->stream));
    Dd acc{0.0, 0.0};
    for (double p : parts) acc = dd_add(acc, p);
    *out = sqrt(dd_value(acc));
  }
  HS_API_END
}

hs_status hs_cg_solve(hs_ctx* c, const hs_matrix* m, const double* d_rhs,
                      const hs_cg_params* p, double* d_x, hs_cg_stats* st,
                      double* trace) {
  HS_API_BEGIN
  HS_REQUIRE(c && m && d_rhs && p && d_x && st, HS_ERR_CONFIG, "null pointer");
  HS_REQUIRE(m->ctx == c, HS_ERR_CONFIG, "matrix belongs to another context");
  HS_CUDA(cudaSetDevice(c->device));
  std::memset(st, 0, sizeof(*st));
  cg_run(c, m, d_rhs, p, d_x, st, trace);  // sets compute_ms (exit diagnostic excluded)
  st->wall_ms = st->compute_ms;
  HS_API_END
}

hs_status hs_solve_cg_host(hs_ctx* c, size_t n, size_t b, const double* a,
                           const double* rhs, const hs_cg_params* p, double* x,
                           hs_cg_stats* st, double* trace) {
  HS_API_BEGIN
  HS_REQUIRE(c && a && rhs && p && x && st, HS_ERR_CONFIG, "null pointer");
  HS_REQUIRE(p->eps > 0.0, HS_ERR_CONFIG, "eps must be positive");
  HS_CUDA(cudaSetDevice(c->device));
  std::memset(st, 0, sizeof(*st));
  // device storage cached by the context across calls (allocated once)
  hs_matrix* m = cached_matrix(c, 0, n, b);
  const size_t pn = (size_t)ceil_div(n, b) * b;
  double* d_rhs = ctx_vec(c, 0, pn);
  double* d_x = ctx_vec(c, 1, pn);
  {
    // wall = initial transfer + solve + result download; compute = the
    // solve; the exit residual diagnostic is outside both
    // (cg_solver.cpp:232-234, 354-356)
    const auto tt = std::chrono::steady_clock::now();
    hs_status s = hs_matrix_upload(m, a);
    if (s != HS_OK) throw Failure{s, hs_last_error()};
    HS_CUDA(cudaMemcpyAsync(d_rhs, rhs, pn * sizeof(double),
                            cudaMemcpyHostToDevice, c->stream));
    HS_CUDA(cudaStreamSynchronize(c->stream));
    double xfer = ms_since(tt);
    cg_run(c, m, d_rhs, p, d_x, st, trace);
    const auto t2 = std::chrono::steady_clock::now();
    HS_CUDA(cudaMemcpyAsync(x, d_x, pn * sizeof(double), cudaMemcpyDeviceToHost,
                            c->stream));
    HS_CUDA(cudaStreamSynchronize(c->stream));
    xfer += ms_since(t2);
    st->transfer_ms = xfer;
    st->wall_ms = xfer + st->compute_ms;
  }
  HS_API_END
}

}  // extern "C"

namespace hs {
// y = A x, full length on every rank: the single-rank SYMV, or (world > 1,
// block-cyclic) each rank's owned-tile partial, all-gathered and summed in
// rank order (identical on every rank; hs_solve_spd_refine)
void symv_full(hs_ctx* c, const hs_matrix* m, const double* x, double* y) {
  if (c->world == 1) {
    symv_local(c, m, x, y);
    return;
  }
  HS_REQUIRE(m->layout == 1, HS_ERR_CONFIG, "multi-rank SYMV needs a block-cyclic matrix");
  const int64_t pn = (int64_t)m->N * (int64_t)m->b;
  const size_t sz[1] = {(size_t)pn * c->world * sizeof(double)};
  void* ws[1];
  ctx_workspace(c, 0, sz, 1, ws);
  double* gath = static_cast<double*>(ws[0]);
  const int b = (int)m->b;
  cyclic_partial_symv_kernel<<<dim3((b + 31) / 32, (unsigned)m->N), 256, 0, c->stream>>>(
      m->d, m->d_lpos, x, y, b, (int64_t)m->N);
  HS_CUDA(cudaGetLastError());
  launch_count(c);
  c->step = -1;
  comm_allgather(c, y, gath, (size_t)pn, LK_RESULT);
  rank_sum_kernel<<<592, 256, 0, c->stream>>>(gath, y, pn, c->world);
  HS_CUDA(cudaGetLastError());
  launch_count(c);
}
}  // namespace hs

#ifdef HS_SYMV_TIMING
// debug builds only: per-launch SYMV (min CTA start, max CTA end) globaltimer
// stamps; reset clears them and sets the per-CTA printf switch
extern "C" int hs_debug_fin_ts(unsigned long long* out, int count, int reset) {
  if (reset) {
    static unsigned long long init[4096][5];
    for (int k = 0; k < 4096; ++k)
      init[k][0] = ~0ull, init[k][1] = init[k][2] = init[k][3] = init[k][4] = 0;
    return (int)cudaMemcpyToSymbol(hs::g_fin_ts, init, sizeof(init));
  }
  return (int)cudaMemcpyFromSymbol(out, hs::g_fin_ts, (size_t)count * 5 * sizeof(unsigned long long));
}

extern "C" int hs_debug_symv_fin_end(unsigned long long* out, int count, int reset) {
  if (reset) {
    static unsigned long long init[4096];
    return (int)cudaMemcpyToSymbol(hs::g_symv_fin_end, init, sizeof(init));
  }
  return (int)cudaMemcpyFromSymbol(out, hs::g_symv_fin_end, (size_t)count * sizeof(unsigned long long));
}

extern "C" int hs_debug_tail_ts(unsigned long long* out, int count, int reset) {
  if (reset) {
    static unsigned long long init[4096][7];
    for (int k = 0; k < 4096; ++k)
      for (int i = 0; i < 7; ++i) init[k][i] = (i == 0 || i == 6) ? ~0ull : 0ull;
    return (int)cudaMemcpyToSymbol(hs::g_tail_ts, init, sizeof(init));
  }
  return (int)cudaMemcpyFromSymbol(out, hs::g_tail_ts, (size_t)count * 7 * sizeof(unsigned long long));
}

extern "C" int hs_debug_tail_cta(unsigned long long* out) {
  return (int)cudaMemcpyFromSymbol(out, hs::g_tail_cta, sizeof(hs::g_tail_cta));
}

extern "C" int hs_debug_symv_ts(unsigned long long* out, int count, int reset, int print) {
  if (reset) {
    static unsigned long long init[4096][2];
    for (int k = 0; k < 4096; ++k) {
      init[k][0] = ~0ull;
      init[k][1] = 0;
    }
    cudaMemcpyToSymbol(hs::g_symv_ts, init, sizeof(init));
    cudaMemcpyToSymbol(hs::g_symv_ts_print, &print, sizeof(int));
    return 0;
  }
  return (int)cudaMemcpyFromSymbol(out, hs::g_symv_ts, (size_t)count * 2 * sizeof(unsigned long long));
}
#endif
