// FP64-accurate GEMM update C -= P Q^T on the sm_100a INT8 tensor cores
// (Ozaki scheme I), for the Cholesky trailing update (reference
// block_kernels.cpp:39-57 gemm_update / syrk_update).
//
// sm_100a has no FP64 tcgen05 kind; its FP64 path is warp-level DMMA at
// ~35 TF/s. The INT8 tensor cores run 4.5 POPS dense, and an FP64 product can
// be rebuilt exactly from INT8 products:
//
//   * slicing (oz_slice_kernel): each operand row r gets an exponent e_r
//     (max_c |x_rc| * 2^-e_r in [0.5, 1)) and s signed 8-bit slices d_1..d_s
//     with x = 2^e_r * sum_p d_p 2^(-6-7(p-1)) + O(2^(e_r - 7s - 1)):
//     d_1 = rint(x 2^(6-e)), then repeatedly t = 128 * remainder,
//     d = rint(t) -- every step exact in FP64, |d_p| <= 64.
//   * products (oz_gemm_kernel): for each slice pair with p + q <= s + 1, an
//     INT8 x INT8 -> INT32 tcgen05.mma accumulates exactly into the TMEM
//     accumulator of group g = p + q (all pairs of a group share the weight
//     2^(-12-7(g-2)); |group sum| <= 8 * K * 64^2 = 2^24 for K = 512). Up to
//     four pairs (p, q..q+3) go out as one N = 256 MMA (see the stage layout).
//   * epilogue: the group sums are folded exactly in int64 (groups 0-3 and
//     4-7, each < 2^46), converted without I2F (2^52 + 2^51 trick),
//     C -= 2^(e_r + e_c) (2^-33 hi + 2^-61 lo) with one FP64 rounding (the
//     power of two applied by exponent arithmetic), read-modify-write of the
//     output block straight from registers.
//
// Dropped pairs (p + q > s + 1) and the slicing tail bound the error per
// element by ~2^(-7s+12) * 2^(e_r+e_c) * K / 2^7 -- for s = 8 at or below the
// worst-case FP64 GEMM rounding bound 2^-53 * K * 2^(e_r+e_c).
//
// Kernel shape: one CTA = 128 output rows x 64 columns, the whole K; all
// s <= 8 group accumulators live in TMEM at once (8 x 64 = 512 columns).
// Persistent with bounded item counts (the Cholesky panel stream must be
// able to interleave), warp-specialized: warp 0 lane 0 issues TMA (per
// 64-wide K chunk one 3-D box per operand carries all s slices, 64-B
// swizzle, 2-stage ring), warp 1 lane 0 issues tcgen05.mma, warps 2-9 drain
// TMEM (two warps per 32-lane quadrant, 32 columns each) and release it
// before the FP64 work, so the next item's MMAs overlap this epilogue.
#include <cuda.h>
#include <math.h>

#include <algorithm>
#include <cstdlib>
#include <vector>

#include "hs_internal.h"

namespace hs {
namespace oz {

constexpr int M = 128;      // output rows per CTA (TMEM lanes)
constexpr int N = 64;       // output columns per CTA
constexpr int KS = 64;      // K (int8 elements = bytes) per stage: two MMA K steps
constexpr int MAXS = 8;     // max slices (8 groups x 64 columns = 512 TMEM cols)
constexpr int STAGES = 2;
// Slices are stored plane-major ([slice][operand row][K]); a stage holds, for
// each slice, the rows' next 64 K bytes (64-B swizzle rows: half the TMA
// row requests of 32-B rows), slices stacked along the row axis. The B slices q..q+3 then form one contiguous 256-row
// K-major operand, so A_p x [B_q .. B_q+3]^T is a single N = 256 MMA whose
// four 64-column results land in the accumulators of groups p+q .. p+q+3 --
// consecutive TMEM columns. 12 MMAs per K step cover all 36 pairs (s = 8).
constexpr int ROWB = KS;                  // bytes per swizzled smem row
constexpr int A_SLICE = M * ROWB;         // 8 KB
constexpr int B_SLICE = N * ROWB;         // 4 KB
constexpr int A_STAGE = MAXS * A_SLICE;   // 32 KB
constexpr int B_STAGE = MAXS * B_SLICE;   // 16 KB
constexpr int STAGE = A_STAGE + B_STAGE;
constexpr int SMEM = STAGES * STAGE + 1024 + 1024;
// warp roles: 0 TMA producer, 1 MMA issuer, 2-9 epilogue (two warps per
// TMEM lane quadrant, 32 output columns each)
constexpr int EPI_WARP0 = 2, EPI_WARPS = 8;
constexpr int THREADS = (EPI_WARP0 + EPI_WARPS) * 32;
constexpr int32_t NONFINITE = -100000;   // row exponent sentinel (NaN / Inf row)

enum Mode : int {
  BATCH = 0,     // C_t -= P_t Q_t^T over `count` contiguous tile triples
  CHOL_COL = 1,  // Cholesky column j: A_i,j+1 -= L_ij L_j+1,j^T, i > j
  CHOL_REST = 2,  // Cholesky column j: A_ik -= L_ij L_kj^T, j + 2 <= k <= i
  CHOL_LIST = 3   // distributed Cholesky column j: the listed owned (i, k)
};

struct Args {
  int mode;
  double* C;            // BATCH: output tiles; CHOL: packed tiles (local)
  const int32_t* EA;    // row exponents of the A operand rows
  const int32_t* EB;    // row exponents of the B operand rows
  int b, s;
  int K;                // operand width (K) per slice row: b, or 2b for column pairs
  int lower_only;       // BATCH: SYRK-style lower-triangle update
  int64_t count;        // BATCH: number of (C, P, Q) triples
  int64_t j, tile_lo;   // CHOL: panel-row origin (rows of tile i at (i-j-1) b), first local tile
  int64_t kk;           // CHOL_COL: the tile column; CHOL_REST: first tile column
  const int32_t* pairs;  // CHOL_LIST: (i, k) pairs of this launch
  const int64_t* lpos;   // CHOL_LIST: packed tile -> local slot (2D block-cyclic)
  const int32_t* status;  // optional: non-zero -> skip (factorization failed)
  long long* prof;        // optional phase timestamps (tools/oz_bench.py --phases)
};

// prof layout: [cta][tile < 64][8] globaltimer stamps
__device__ __forceinline__ void prof_stamp(long long* prof, int64_t lt, int k) {
  if (prof && lt < 64) {
    long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    prof[((int64_t)blockIdx.x * 64 + lt) * 8 + k] = t;
  }
}

// ---------------------------------------------------------------------------
// slicing: one warp per operand row; lane handles 4 consecutive elements
// per step so every int8 slice row is written with 32-bit stores.

// Operand rows (K = b, or 2b for a column pair) of `rows` rows:
//   colA < 0: contiguous rows of X (K = b);
//   colA >= 0: row r of panel tile t is row r of packed tile (jb + 1 + t, colA)
//   (tile index tri(i, col) - tile_lo), followed, when colB >= 0, by row r of
//   tile (jb + 1 + t, colB): the concatenated operand of a two-column update.
// Output: exponent E[row] and S[p][row][K] for p < s (plane = plane_rows K).
__global__ void __launch_bounds__(256)
    slice_kernel(const double* __restrict__ X, int64_t rows, int b, int s,
                 int8_t* __restrict__ S, int32_t* __restrict__ E, int64_t plane_rows,
                 int64_t colA, int64_t colB, int64_t jb, int64_t tile_lo,
                 const int32_t* status) {
  if (status && *status) return;
  const int64_t row = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= rows) return;
  const int64_t t = row / b, r = row % b;
  const int K = colB >= 0 ? 2 * b : b;
  const double* seg0;
  const double* seg1 = nullptr;
  if (colA < 0) {
    seg0 = X + row * (int64_t)b;
  } else {
    const int64_t i = jb + 1 + t;
    seg0 = X + ((tri(i, colA) - tile_lo) * b + r) * (int64_t)b;
    if (colB >= 0) seg1 = X + ((tri(i, colB) - tile_lo) * b + r) * (int64_t)b;
  }
  auto at = [&](int c) { return c < b ? seg0[c] : seg1[c - b]; };
  double mx = 0.0;
  bool finite = true;
  for (int c = lane; c < K; c += 32) {
    const double v = at(c);
    finite &= isfinite(v);
    mx = fmax(mx, fabs(v));
  }
  for (int o = 16; o; o >>= 1) {
    mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    finite = __all_sync(0xffffffffu, finite);
  }
  const int e = (mx > 0.0) ? ilogb(mx) + 1 : 0;
  if (lane == 0) E[row] = finite ? e : NONFINITE;
  // plane-major: slice p of this row at S + (p * plane_rows + row) * K
  int8_t* base = S + row * (int64_t)K;
  const int64_t pstride = plane_rows * (int64_t)K;
  for (int c0 = lane * 4; c0 < K; c0 += 128) {
    double rem[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) rem[u] = finite ? ldexp(at(c0 + u), 6 - e) : 0.0;
    for (int p = 0; p < s; ++p) {
      uint32_t w = 0;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const double d = rint(rem[u]);
        rem[u] = (rem[u] - d) * 128.0;
        w |= (uint32_t)(uint8_t)(int8_t)(int)d << (8 * u);
      }
      *reinterpret_cast<uint32_t*>(base + p * pstride + c0) = w;
    }
  }
}

// ---------------------------------------------------------------------------
// tcgen05 / TMA primitives

__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int c0,
                                            int c1, int c2, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_"
      "tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}

// K-major operand tile in shared memory, 64-byte swizzle (TMA
// CU_TENSOR_MAP_SWIZZLE_64B): rows of 64 B, 8-row atoms of 512 B; the start
// address may sit 32 B into the row (second MMA K step).
__device__ __forceinline__ uint64_t sdesc_sw64(uint32_t saddr) {
  uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFF);  // start address
  d |= (uint64_t)1 << 16;                           // LBO (unused, swizzled K-major)
  d |= (uint64_t)(512 >> 4) << 32;                  // SBO: next 8-row atom
  d |= (uint64_t)1 << 46;                           // descriptor version (sm_100)
  d |= (uint64_t)4 << 61;                           // layout: SWIZZLE_64B
  return d;
}

// kind::i8 instruction descriptor: s8 x s8 -> s32, K-major A and B.
__host__ __device__ constexpr uint32_t idesc_i8(int m, int n) {
  return (2u << 4)                       // D format s32
         | (1u << 7) | (1u << 10)        // A, B signed int8
         | ((uint32_t)(n >> 3) << 17)    // N
         | ((uint32_t)(m >> 4) << 24);   // M
}

__device__ __forceinline__ void mma_i8(uint32_t tmem_d, uint64_t da, uint64_t db,
                                       uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(accumulate)
      : "memory");
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}

// 16 consecutive TMEM columns of this thread's lane -> registers (no wait)
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, int32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,"
      "%12,%13,%14,%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]),
        "=r"(v[6]), "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]),
        "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
}
// 32 consecutive TMEM columns of this thread's lane -> registers (no wait)
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, int32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,"
      "%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,"
      "%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]),
        "=r"(v[6]), "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]),
        "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]),
        "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
        "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]),
        "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// -x * 2^e by exponent arithmetic (integer ops only; FP64 pipe untouched):
// exact whenever x and the result are normal, ldexp otherwise.
__device__ __forceinline__ double neg_scale2(double x, int e) {
  const long long bits = __double_as_longlong(x);
  const int ex = (int)((bits >> 52) & 0x7ff);
  if (ex == 0 || ex + e <= 0 || ex + e >= 0x7ff) return -ldexp(x, e);  // 0, subnormal, range
  return __longlong_as_double((bits + ((long long)e << 52)) ^ (long long)0x8000000000000000ull);
}

// 2^e as a double (normal range; ldexp outside it)
__device__ __forceinline__ double pow2(int e) {
  return (e > -1023 && e < 1024) ? __longlong_as_double((long long)(e + 1023) << 52)
                                 : ldexp(1.0, e);
}

// ---------------------------------------------------------------------------
// one output sub-block: decoded item

struct Item {
  int a_row, b_row; // first operand row (global row of the slice buffers)
  int a_off, b_off; // row offsets inside their b x b tiles
  int64_t ea, eb;   // exponent index of the first A / B row
  double* c;        // output (row-major, ld = b)
  bool lower;       // mask to the lower triangle (col <= row) of the tile
  bool skip;
};

__device__ __forceinline__ Item decode_item(const Args& g, int64_t item) {
  const int fm = g.b / M, fn = g.b / N;
  const int64_t u = item / (fm * fn);
  const int sb = (int)(item % (fm * fn));
  const int mb = sb / fn, nb = sb % fn;
  const int64_t bb = (int64_t)g.b * g.b;
  Item it;
  it.a_off = mb * M;
  it.b_off = nb * N;
  bool diag;
  if (g.mode == BATCH) {
    it.a_row = (int)(u * g.b + mb * M);
    it.b_row = (int)(u * g.b + nb * N);
    it.c = g.C + u * bb + (int64_t)mb * M * g.b + nb * N;
    diag = g.lower_only != 0;
  } else {
    // trailing tile (i, k) of column j; panel rows of tile i start at
    // (i - j - 1) b in the slice buffer (gemm_update / syrk_update,
    // block_kernels.cpp:39-57)
    int64_t i, k;
    if (g.mode == CHOL_COL) {
      i = g.kk + u;
      k = g.kk;
    } else if (g.mode == CHOL_LIST) {
      i = g.pairs[2 * u];
      k = g.pairs[2 * u + 1];
    } else {
      const int64_t ii = tile_row(u);
      i = g.kk + ii;
      k = g.kk + (u - tri(ii, 0));
    }
    it.a_row = (int)((i - g.j - 1) * g.b + mb * M);
    it.b_row = (int)((k - g.j - 1) * g.b + nb * N);
    const int64_t slot = g.mode == CHOL_LIST ? g.lpos[tri(i, k)] : tri(i, k) - g.tile_lo;
    it.c = g.C + slot * bb + (int64_t)mb * M * g.b + nb * N;
    diag = i == k;
  }
  it.ea = it.a_row;
  it.eb = it.b_row;
  // sub-block rows [mb*M, +M), cols [nb*N, +N) of the tile
  it.lower = diag && (nb * N + N - 1 > mb * M);
  it.skip = diag && (nb * N > mb * M + M - 1);
  return it;
}

// Persistent, warp-specialized: each CTA walks items blockIdx.x,
// blockIdx.x + gridDim.x, ...; the smem ring runs ahead across items, and the
// epilogue of item i (TMEM -> registers -> FP64 read-modify-write of C)
// overlaps the loads and MMAs of item i + 1 -- the accumulators are released
// as soon as they are read, before the FP64 work and the global update.
template <int S>
__global__ void __launch_bounds__(THREADS, 1)
    gemm_kernel(const __grid_constant__ CUtensorMap mapA,
                const __grid_constant__ CUtensorMap mapB, Args g, int64_t items) {
  if (g.status && *g.status) return;
  const int nk = g.K / KS;

  extern __shared__ __align__(1024) unsigned char raw[];
  // align by offsetting the shared pointer (a uintptr_t round trip would
  // make the epilogue's exponent reads generic loads)
  unsigned char* sm = raw + ((1024u - (smem_u32(raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + STAGES * STAGE);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 1);
  int32_t* ebs = reinterpret_cast<int32_t*>(tempty + 2);  // [2][N] column exponents
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    mbar_init(tfull, 1);
    mbar_init(tempty, EPI_WARPS);
    fence_mbar_init();
  }
  if (warp == 0) {  // whole warp: allocate all 512 TMEM columns
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                     smem_u32(tmem_slot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // ---- TMA producer: all S slices of the A rows and B rows per K chunk
      const uint32_t bytes = (uint32_t)(S * (M + N) * ROWB);
      int64_t kg = 0;
      for (int64_t item = blockIdx.x; item < items; item += gridDim.x) {
        const Item it = decode_item(g, item);
        if (it.skip) continue;
        for (int kc = 0; kc < nk; ++kc, ++kg) {
          const int st = (int)(kg % STAGES);
          if (kg >= STAGES) mbar_wait(&empty[st], (uint32_t)((kg / STAGES) - 1) & 1);
          unsigned char* sa = sm + st * STAGE;
          mbar_arrive_expect_tx(&full[st], bytes);
          tma_load_3d(sa, &mapA, kc * KS, it.a_row, 0, &full[st]);
          tma_load_3d(sa + A_STAGE, &mapB, kc * KS, it.b_row, 0, &full[st]);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---- MMA issuer: pairs (p, q), p + q < S (0-based) into group p + q;
      // q in chunks of up to 4 per N <= 256 MMA; fully unrolled
      int64_t kg = 0, lt = 0;
      for (int64_t item = blockIdx.x; item < items; item += gridDim.x) {
        const Item it = decode_item(g, item);
        if (it.skip) continue;
        prof_stamp(g.prof, lt, 0);
        if (lt > 0) mbar_wait(tempty, (uint32_t)(lt - 1) & 1);  // accumulators drained
        tc_fence_after();
        prof_stamp(g.prof, lt, 1);
        for (int kc = 0; kc < nk; ++kc, ++kg) {
          const int st = (int)(kg % STAGES);
          mbar_wait(&full[st], (uint32_t)(kg / STAGES) & 1);
          tc_fence_after();
#pragma unroll
          for (int ks = 0; ks < KS / 32; ++ks) {
            const uint64_t da = sdesc_sw64(smem_u32(sm + st * STAGE) + ks * 32);
            const uint64_t db = sdesc_sw64(smem_u32(sm + st * STAGE + A_STAGE) + ks * 32);
#pragma unroll
            for (int p = 0; p < S; ++p) {
              // the p = 0 MMAs touch every group first: they overwrite at
              // the first K step, everything else accumulates
              const uint32_t acc = (kc > 0 || ks > 0 || p > 0) ? 1u : 0u;
#pragma unroll
              for (int q0 = 0; q0 < S - p; q0 += 4) {
                const int len = (S - p - q0) < 4 ? (S - p - q0) : 4;
                mma_i8(tmem + (uint32_t)((p + q0) * N), da + (uint64_t)((p * A_SLICE) >> 4),
                       db + (uint64_t)((q0 * B_SLICE) >> 4), idesc_i8(M, N * len), acc);
              }
            }
          }
          mma_commit(&empty[st]);  // frees the stage when these MMAs complete
        }
        mma_commit(tfull);
        prof_stamp(g.prof, lt, 2);
        ++lt;
      }
    }
  } else if (warp >= EPI_WARP0) {
    // ---- epilogue: warp quadrant qd = warp % 4 -> TMEM lanes 32 qd.., rows;
    // half h = (warp - EPI_WARP0) / 4 -> columns 32 h .. 32 h + 31
    const int qd = warp & 3, half = (warp - EPI_WARP0) >> 2;
    const int row = qd * 32 + lane;
    const uint32_t lane_addr = tmem + ((uint32_t)(qd * 32) << 16) + (uint32_t)(half * 32);
    const bool issuer = threadIdx.x == EPI_WARP0 * 32;
    const int et = threadIdx.x - EPI_WARP0 * 32;  // 0 .. 255
    int64_t lt = 0;
    for (int64_t item = blockIdx.x; item < items; item += gridDim.x) {
      const Item it = decode_item(g, item);
      if (it.skip) continue;
      const int32_t ea = g.EA[it.ea + row];
      // column exponents of this item, staged while the MMAs run (double
      // buffered: a slow warp may still read the previous item's)
      int32_t* eb_s = ebs + (lt & 1) * N;
      if (et < N) eb_s[et] = g.EB[it.eb + et];
      if (issuer) prof_stamp(g.prof, lt, 3);
      mbar_wait(tfull, (uint32_t)lt & 1);
      tc_fence_after();
      if (issuer) prof_stamp(g.prof, lt, 4);
      // drain: per 16-column half, fold the groups exactly in int64 (groups
      // 0-3 -> hi, 4-7 -> lo, each < 2^46), convert both with the 2^52 + 2^51
      // magic-number trick (no I2F: the conversion pipe was the drain's
      // bottleneck), acc = 2^-33 hi + 2^-61 lo (one FP64 rounding); then hand
      // the accumulators back to the MMA warp
      constexpr int HG = S < 4 ? S : 4, LG = S > 4 ? S - 4 : 0;
      const double whi = pow2(-12 - 7 * (HG - 1));
      const double wlo = pow2(-12 - 7 * (4 + LG - 1));
      double acc[32];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        long long hi[16], lo[16];
#pragma unroll
        for (int c = 0; c < 16; ++c) hi[c] = lo[c] = 0;
#pragma unroll
        for (int grp = 0; grp < S; ++grp) {
          int32_t v[16];
          tmem_ld16(lane_addr + (uint32_t)(grp * N + h * 16), v);
          tmem_wait_ld();
#pragma unroll
          for (int c = 0; c < 16; ++c) {
            if (grp < 4) hi[c] = (hi[c] << 7) + v[c];
            else lo[c] = (lo[c] << 7) + v[c];
          }
        }
        constexpr long long kMagic = 0x4338000000000000ll;  // 2^52 + 2^51
        const double kMagicD = 6755399441055744.0;
#pragma unroll
        for (int c = 0; c < 16; ++c) {
          const double dh = __longlong_as_double(hi[c] + kMagic) - kMagicD;
          const double dl = __longlong_as_double(lo[c] + kMagic) - kMagicD;
          acc[h * 16 + c] = fma(dl, wlo, dh * whi);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(tempty);
      if (issuer) prof_stamp(g.prof, lt, 5);
      const bool bad_row = ea == NONFINITE;
      named_bar_sync(1, EPI_WARPS * 32);  // every thread's exponents are in eb_s
      if (issuer) prof_stamp(g.prof, lt, 7);
      const double qnan = __longlong_as_double(0x7ff8000000000000ll);
      // write-back straight from registers: this CTA owns the output block,
      // so a plain read-modify-write of the thread's 32-column row segment
      // (16-B accesses). Measured faster than staging through shared memory
      // (a smem transpose + coalesced RMW, or TMA tensor reduce-adds): the
      // tensor cores' operand reads keep the smem/L1 datapath busy, and every
      // extra smem pass of the epilogue stretches it.
      double* crow = it.c + (int64_t)row * g.b + half * 32;
      const int grow = it.a_off + row;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        double2 cur[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) cur[u] = reinterpret_cast<const double2*>(crow)[h * 8 + u];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int c = h * 16 + 2 * u, cc = half * 32 + c;
          const int32_t eb0 = eb_s[cc], eb1 = eb_s[cc + 1];
          const double d0 = (bad_row || eb0 == NONFINITE) ? qnan : neg_scale2(acc[c], ea + eb0);
          const double d1 =
              (bad_row || eb1 == NONFINITE) ? qnan : neg_scale2(acc[c + 1], ea + eb1);
          double2 v = cur[u];
          if (!it.lower || it.b_off + cc <= grow) v.x += d0;
          if (!it.lower || it.b_off + cc + 1 <= grow) v.y += d1;
          reinterpret_cast<double2*>(crow)[h * 8 + u] = v;
        }
      }
      if (issuer) prof_stamp(g.prof, lt, 6);
      ++lt;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem)
                 : "memory");
}

template <int S>
static void launch_gemm_s(hs_ctx* c, cudaStream_t st, const CUtensorMap& ma,
                          const CUtensorMap& mb, const Args& g,
                          int64_t items) {
  static std::atomic<uint64_t> attr{0};
  HS_CUDA(smem_attr_once(gemm_kernel<S>, SMEM, attr));
  // Bounded persistence: each CTA walks ~ipc items (strided by the grid, so
  // co-resident CTAs work on neighbouring items), then retires. A CTA that
  // owned its SM for the whole update would lock the Cholesky's
  // high-priority panel stream out of the GPU; retiring every few tiles lets
  // the block scheduler slip panel CTAs in.
  static const int ipc = [] {
    const char* e = getenv("HS_OZ_ITEMS_PER_CTA");
    return e ? std::max(1, atoi(e)) : 16;
  }();
  const int64_t grid = std::max<int64_t>(
      std::min<int64_t>(items, c->num_sms), ceil_div(items, ipc));
  gemm_kernel<S><<<(unsigned)grid, THREADS, SMEM, st>>>(ma, mb, g, items);
  HS_CUDA(cudaGetLastError());
  launch_count(c);
}

static void launch_gemm(hs_ctx* c, cudaStream_t st, const CUtensorMap& ma,
                        const CUtensorMap& mb, const Args& g,
                        int64_t items) {
  if (items <= 0) return;
  switch (g.s) {
    case 1: launch_gemm_s<1>(c, st, ma, mb, g, items); break;
    case 2: launch_gemm_s<2>(c, st, ma, mb, g, items); break;
    case 3: launch_gemm_s<3>(c, st, ma, mb, g, items); break;
    case 4: launch_gemm_s<4>(c, st, ma, mb, g, items); break;
    case 5: launch_gemm_s<5>(c, st, ma, mb, g, items); break;
    case 6: launch_gemm_s<6>(c, st, ma, mb, g, items); break;
    case 7: launch_gemm_s<7>(c, st, ma, mb, g, items); break;
    default: launch_gemm_s<8>(c, st, ma, mb, g, items); break;
  }
}

// 3-D map over the slice planes [slice][row][K]: box 64 B x box_rows x s.
static CUtensorMap slice_map(const int8_t* base, int K, int64_t rows, int box_rows, int s) {
  cuuint64_t dims[3] = {(cuuint64_t)K, (cuuint64_t)std::max<int64_t>(rows, 1), (cuuint64_t)MAXS};
  cuuint64_t strides[2] = {(cuuint64_t)K, (cuuint64_t)K * std::max<int64_t>(rows, 1)};
  cuuint32_t box[3] = {(cuuint32_t)KS, (cuuint32_t)box_rows, (cuuint32_t)s};
  return make_tensor_map(CU_TENSOR_MAP_DATA_TYPE_UINT8, base, 3, dims, strides, box,
                         CU_TENSOR_MAP_SWIZZLE_64B);
}

}  // namespace oz

// Slice `tiles` consecutive b x b FP64 tiles (tiles * b operand rows) into
// int8 slice planes ([slice][row][K], plane = plane_rows * b bytes), plus
// per-row exponents.
void oz_slice(hs_ctx* c, cudaStream_t st, const double* X, int64_t tiles, int b, int s,
              int8_t* S, int32_t* E, int64_t plane_rows, int64_t colA, int64_t colB,
              int64_t jb, int64_t tile_lo, const int32_t* status) {
  const int64_t rows = tiles * b;
  if (rows <= 0) return;
  oz::slice_kernel<<<(unsigned)ceil_div(rows, 8), 256, 0, st>>>(X, rows, b, s, S, E,
                                                                 plane_rows, colA, colB, jb,
                                                                 tile_lo, status);
  HS_CUDA(cudaGetLastError());
  launch_count(c);
}

// ---- Cholesky trailing update on the INT8 tensor cores ---------------------

OzPanel::~OzPanel() {
  for (int k = 0; k < 2; ++k) {
    cudaFree(S[k]);
    cudaFree(E[k]);
    cudaFree(SJ[k]);
    cudaFree(EJ[k]);
  }
}

void OzPanel::init(int b_, int64_t N_, int s_, bool pairs) {
  b = b_;
  s = s_;
  rows = std::max<int64_t>(N_ - 1, 1) * b;
  // buffers are kept across factorizations (a cudaMalloc / cudaFree of the
  // ~0.8 GB at n = 32768 per call cost tens of ms): grow only
  const size_t need_s = (size_t)rows * b * oz::MAXS;
  const size_t need_e = (size_t)rows * sizeof(int32_t);
  const size_t need_sj = pairs ? (size_t)rows * 2 * b * oz::MAXS : 0;
  for (int k = 0; k < 2; ++k) {
    if (need_s > cap_s) {
      cudaFree(S[k]);
      S[k] = nullptr;
      HS_CUDA(cudaMalloc(&S[k], need_s));
    }
    if (need_e > cap_e) {
      cudaFree(E[k]);
      cudaFree(EJ[k]);
      E[k] = EJ[k] = nullptr;
      HS_CUDA(cudaMalloc(&E[k], need_e));
      HS_CUDA(cudaMalloc(&EJ[k], need_e));
    }
    if (need_sj > cap_sj) {
      cudaFree(SJ[k]);
      SJ[k] = nullptr;
      HS_CUDA(cudaMalloc(&SJ[k], need_sj));
    }
  }
  cap_s = std::max(cap_s, need_s);
  cap_e = std::max(cap_e, need_e);
  cap_sj = std::max(cap_sj, need_sj);
}

OzPanel& ctx_oz_panel(hs_ctx* c) {
  if (!c->oz_panel) c->oz_panel = new OzPanel;
  return *c->oz_panel;
}

// Slices the panel tiles (i, j), i > j, of column j into buffer j & 1.
void OzPanel::slice(hs_ctx* c, cudaStream_t st, const double* A, int64_t tile_lo, int64_t N,
                    int64_t j, const int32_t* status) {
  const int64_t t = N - 1 - j;
  oz_slice(c, st, A, t, b, s, S[j & 1], E[j & 1], rows, j, -1, j, tile_lo, status);
}

// Joint slices of the column pair (j0, j0 + 1): operand rows
// [L_i,j0 | L_i,j0+1] (K = 2b, one exponent per row) of the tiles
// i >= j0 + 2, into pair buffer (j0 / 2) & 1.
void OzPanel::slice_pair(hs_ctx* c, cudaStream_t st, const double* A, int64_t tile_lo,
                         int64_t N, int64_t j0, const int32_t* status) {
  const int64_t t = N - 2 - j0;
  const int k = (int)((j0 / 2) & 1);
  oz_slice(c, st, A, t, b, s, SJ[k], EJ[k], rows, j0, j0 + 1, j0 + 1, tile_lo, status);
}

static void launch_update(hs_ctx* c, cudaStream_t st, const int8_t* S, const int32_t* E,
                          int b, int K, int s, int64_t rows, double* A, int64_t tile_lo,
                          int64_t jb, int mode, int64_t kk, int64_t tiles,
                          const int32_t* status) {
  if (tiles <= 0) return;
  const int fm = b / oz::M, fn = b / oz::N;
  const CUtensorMap ma = oz::slice_map(S, K, rows, oz::M, s);
  const CUtensorMap mb = oz::slice_map(S, K, rows, oz::N, s);
  oz::Args g{};
  g.mode = mode;
  g.C = A;
  g.EA = g.EB = E;
  g.b = b;
  g.K = K;
  g.s = s;
  g.j = jb;
  g.kk = kk;
  g.tile_lo = tile_lo;
  g.status = status;
  oz::launch_gemm(c, st, ma, mb, g, tiles * fm * fn);
}

// A_ik -= L_ij L_kj^T for the tiles of column j: `col` selects k == j + 1
// (the lookahead column), else j + 2 <= k <= i.
void OzPanel::update(hs_ctx* c, cudaStream_t st, double* A, int64_t tile_lo,
                     int64_t local_tiles, int64_t N, int64_t j, bool col,
                     const int32_t* status) {
  (void)local_tiles;
  const int64_t t = N - 1 - j;
  launch_update(c, st, S[j & 1], E[j & 1], b, b, s, rows, A, tile_lo, j,
                col ? oz::CHOL_COL : oz::CHOL_REST, col ? j + 1 : j + 2,
                col ? t : (t - 1) * t / 2, status);
}

// A_ik -= [L_i,j0 L_i,j0+1] [L_k,j0 L_k,j0+1]^T (K = 2b): `col` = the single
// tile column k == kk, else every k >= kk.
void OzPanel::update_pair(hs_ctx* c, cudaStream_t st, double* A, int64_t tile_lo, int64_t N,
                          int64_t j0, bool col, int64_t kk, const int32_t* status) {
  const int64_t t = N - kk;  // tile columns kk .. N-1
  const int k = (int)((j0 / 2) & 1);
  launch_update(c, st, SJ[k], EJ[k], b, 2 * b, s, rows, A, tile_lo, j0 + 1,
                col ? oz::CHOL_COL : oz::CHOL_REST, kk, col ? t : t * (t + 1) / 2, status);
}

// Distributed variant: the panel of column j arrives broadcast into a
// contiguous buffer X (tile i at (i - j - 1) b^2); slice it as is.
void OzPanel::slice_contig(hs_ctx* c, cudaStream_t st, const double* X, int64_t N, int64_t j,
                           const int32_t* status) {
  const int64_t t = N - 1 - j;
  oz_slice(c, st, X, t, b, s, S[j & 1], E[j & 1], rows, -1, -1, j, 0, status);
}

// A_ik -= L_ij L_kj^T for `npairs` owned (i, k) of column j (device list),
// output tiles at their 2D block-cyclic local slots.
void OzPanel::update_list(hs_ctx* c, cudaStream_t st, double* A, const int64_t* lpos,
                          int64_t j, const int32_t* pairs, int64_t npairs,
                          const int32_t* status) {
  if (npairs <= 0) return;
  const int fm = b / oz::M, fn = b / oz::N;
  const CUtensorMap ma = oz::slice_map(S[j & 1], b, rows, oz::M, s);
  const CUtensorMap mb = oz::slice_map(S[j & 1], b, rows, oz::N, s);
  oz::Args g{};
  g.mode = oz::CHOL_LIST;
  g.C = A;
  g.EA = g.EB = E[j & 1];
  g.b = b;
  g.K = b;
  g.s = s;
  g.j = j;
  g.pairs = pairs;
  g.lpos = lpos;
  g.status = status;
  oz::launch_gemm(c, st, ma, mb, g, npairs * fm * fn);
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

// test / tuning hook: phase timestamps of the next hs_oz_gemm_tiles call
static long long* g_oz_prof = nullptr;

extern "C" {

void hs_oz_set_profile(void* d_buf) { g_oz_prof = static_cast<long long*>(d_buf); }

hs_status hs_oz_gemm_tiles(hs_ctx* c, double* d_c, const double* d_p, const double* d_q,
                           size_t b, size_t count, int slices, int lower_only) {
  HS_API_BEGIN
  HS_REQUIRE(c && d_c && d_p && d_q, HS_ERR_CONFIG, "null pointer");
  HS_REQUIRE(b % 128 == 0 && b > 0, HS_ERR_CONFIG, "the INT8 path needs b % 128 == 0");
  HS_REQUIRE(slices >= 1 && slices <= oz::MAXS, HS_ERR_CONFIG, "slices must be in [1, 8]");
  HS_CUDA(cudaSetDevice(c->device));
  if (count == 0) return HS_OK;
  const int s = slices;
  const size_t plane = b * b;
  int8_t *sp = nullptr, *sq = nullptr;
  int32_t *ep = nullptr, *eq = nullptr;
  auto release = [&] {
    cudaFree(sp);
    cudaFree(sq);
    cudaFree(ep);
    cudaFree(eq);
  };
  try {
    HS_CUDA(cudaMalloc(&sp, count * oz::MAXS * plane));
    HS_CUDA(cudaMalloc(&sq, count * oz::MAXS * plane));
    HS_CUDA(cudaMalloc(&ep, count * b * sizeof(int32_t)));
    HS_CUDA(cudaMalloc(&eq, count * b * sizeof(int32_t)));
    const int64_t rows = (int64_t)(count * b);
    oz_slice(c, c->stream, d_p, (int64_t)count, (int)b, s, sp, ep, rows, -1, -1, 0, 0, nullptr);
    oz_slice(c, c->stream, d_q, (int64_t)count, (int)b, s, sq, eq, rows, -1, -1, 0, 0, nullptr);
    const CUtensorMap ma = oz::slice_map(sp, (int)b, rows, oz::M, s);
    const CUtensorMap mb = oz::slice_map(sq, (int)b, rows, oz::N, s);
    oz::Args g{};
    g.mode = oz::BATCH;
    g.prof = g_oz_prof;
    g.K = (int)b;
    g.C = d_c;
    g.EA = ep;
    g.EB = eq;
    g.b = (int)b;
    g.s = s;
    g.lower_only = lower_only;
    g.count = (int64_t)count;
    const int64_t items = (int64_t)count * (b / oz::M) * (b / oz::N);
    oz::launch_gemm(c, c->stream, ma, mb, g, items);
    HS_CUDA(cudaStreamSynchronize(c->stream));
  } catch (...) {
    release();
    throw;
  }
  release();
  HS_API_END
}

}  // extern "C"
