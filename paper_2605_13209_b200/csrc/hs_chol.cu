// Tiled right-looking Cholesky + triangular solves on B200
// (reference cholesky_solver.cpp:23-42, 158-254, 275-331).
//
// Per column j of b x b tiles:
//   P stream (high priority, critical path):
//     potrf_tile  L_jj (single CTA, blocked 32-wide)           [K2 potf_block]
//     trtri_tile  W_jj = L_jj^-1 (single CTA)                  [for K3 / K6]
//     tile GEMM   X_i = A_ij W_jj^T  (TRSM as a GEMM)          [K3 trsm_block]
//     copy        A_ij <- X_i
//   U stream (bulk of the flops):
//     tile GEMM   A_ik -= X_i X_k^T, j < k <= i (lower only on i == k)
//                                                          [K4/K5 gemm/syrk]
// with one column of lookahead: the update of tile column j+1 runs first, so
// the P stream factors column j+1 while the rest of column j's update runs.
//
// Tile GEMM: FP64 tensor cores. sm_100a tcgen05 has no f64 kind, so the
// DMMA path is warp-level mma.sync.m8n8k4.f64 (SASS DMMA) fed by TMA
// (cp.async.bulk.tensor, 128-B swizzle) through a 3-stage mbarrier ring with
// a dedicated producer warp. CTA tile 128 x 128, K slice 32, 8 MMA warps of
// 32 x 64. Tiles with b % 128 != 0 use a SIMT FP64 tile kernel.
#include <cuda.h>
#include <math.h>

#include <algorithm>
#include <chrono>
#include <cstring>
#include <vector>

#include "hs_internal.h"

namespace hs {

struct CholFlag {
  int32_t status;  // HS_OK / NOT_SPD / SINGULAR / NUMERICAL
  int32_t pad;
  int64_t col;     // failing column (block row)
  int64_t pivot;   // pivot / diagonal index inside the tile
};

__device__ void raise_flag(CholFlag* f, int status, int64_t col, int64_t piv) {
  if (atomicCAS(&f->status, 0, status) == 0) {
    f->col = col;
    f->pivot = piv;
    __threadfence();
  }
}

// ---------------------------------------------------------------------------
// POTRF of b x b tiles (one CTA per tile). Blocked right-looking, 32-wide
// panels: warp 0 factors the 32x32 diagonal block in shared memory, every
// thread solves one panel row, then a 4x4-register-tiled rank-32 update of
// the trailing lower triangle. Upper triangle untouched (potf_block).

constexpr int PNB = 32;
constexpr int PLD = 33;  // padded leading dimension in shared memory

__global__ void __launch_bounds__(256)
    potrf_tile_kernel(double* base, int64_t stride, int b, CholFlag* flag,
                      int64_t column) {
  if (flag->status) return;
  double* D = base + (int64_t)blockIdx.x * stride;
  extern __shared__ double psm[];
  double* Ds = psm;              // 32 x 33
  double* Ps = psm + PNB * PLD;  // (b) x 33 panel
  __shared__ int bad;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  for (int c0 = 0; c0 < b; c0 += PNB) {
    const int nb = min(PNB, b - c0);
    for (int idx = tid; idx < PNB * PNB; idx += blockDim.x) {
      const int r = idx / PNB, c = idx % PNB;
      Ds[r * PLD + c] =
          (r < nb && c <= r) ? D[(int64_t)(c0 + r) * b + c0 + c] : 0.0;
    }
    if (tid == 0) bad = -1;
    __syncthreads();
    if (warp == 0) {
      for (int p = 0; p < nb; ++p) {
        double d = Ds[p * PLD + p];
        if (!(d > 0.0)) {
          if (lane == 0) bad = c0 + p;
          break;
        }
        d = sqrt(d);
        __syncwarp();
        if (lane == p) Ds[p * PLD + p] = d;
        if (lane > p && lane < nb) Ds[lane * PLD + p] /= d;
        __syncwarp();
        if (lane > p && lane < nb) {
          const double lp = Ds[lane * PLD + p];
          for (int c = p + 1; c <= lane; ++c)
            Ds[lane * PLD + c] = fma(-lp, Ds[c * PLD + p], Ds[lane * PLD + c]);
        }
        __syncwarp();
      }
    }
    __syncthreads();
    if (bad >= 0) {
      if (tid == 0) raise_flag(flag, HS_ERR_NOT_SPD, column, bad);
      return;
    }
    for (int idx = tid; idx < nb * nb; idx += blockDim.x) {
      const int r = idx / nb, c = idx % nb;
      if (c <= r) D[(int64_t)(c0 + r) * b + c0 + c] = Ds[r * PLD + c];
    }
    // panel rows below: x L^T = a  (row-wise forward substitution)
    const int m = b - c0 - nb;
    for (int r = tid; r < m; r += blockDim.x) {
      double* row = D + (int64_t)(c0 + nb + r) * b + c0;
      double x[PNB];
#pragma unroll
      for (int c = 0; c < PNB; ++c) x[c] = c < nb ? row[c] : 0.0;
#pragma unroll
      for (int c = 0; c < PNB; ++c) {
        if (c < nb) {
          double acc = x[c];
#pragma unroll
          for (int k = 0; k < c; ++k) acc = fma(-x[k], Ds[c * PLD + k], acc);
          x[c] = acc / Ds[c * PLD + c];
        }
      }
#pragma unroll
      for (int c = 0; c < PNB; ++c)
        if (c < nb) {
          row[c] = x[c];
          Ps[r * PLD + c] = x[c];
        }
    }
    __syncthreads();
    // trailing lower update, 4x4 micro-tiles
    const int mt = (m + 3) / 4;
    const int ntile = mt * (mt + 1) / 2;
    const int o = c0 + nb;
    for (int u = tid; u < ntile; u += blockDim.x) {
      const int ti = (int)tile_row(u);
      const int tj = u - (int)tri(ti, 0);
      const int r0 = ti * 4, q0 = tj * 4;
      double acc[4][4];
#pragma unroll
      for (int x = 0; x < 4; ++x)
#pragma unroll
        for (int y = 0; y < 4; ++y) acc[x][y] = 0.0;
      for (int k = 0; k < nb; ++k) {
        double a[4], bq[4];
#pragma unroll
        for (int x = 0; x < 4; ++x) {
          a[x] = (r0 + x < m) ? Ps[(r0 + x) * PLD + k] : 0.0;
          bq[x] = (q0 + x < m) ? Ps[(q0 + x) * PLD + k] : 0.0;
        }
#pragma unroll
        for (int x = 0; x < 4; ++x)
#pragma unroll
          for (int y = 0; y < 4; ++y) acc[x][y] = fma(a[x], bq[y], acc[x][y]);
      }
#pragma unroll
      for (int x = 0; x < 4; ++x)
#pragma unroll
        for (int y = 0; y < 4; ++y) {
          const int r = r0 + x, q = q0 + y;
          if (r < m && q <= r) D[(int64_t)(o + r) * b + o + q] -= acc[x][y];
        }
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// TRTRI: W = L^-1 of lower b x b tiles (one CTA per tile), W written full
// (zeros above the diagonal). Row blocks of 32: warp 0 inverts the diagonal
// block in shared memory; each thread owns one column c < r0 of the block
// row: t = L[r0:r0+32, c:r0] W[c:r0, c] (32 accumulators), then
// W[r0:r0+32, c] = -Winv t. Zero / NaN diagonal -> singular_block.

__global__ void __launch_bounds__(256)
    trtri_tile_kernel(const double* lbase, int64_t lstride, double* wbase,
                      int b, CholFlag* flag, int64_t column0) {
  if (flag && flag->status) return;
  const double* L = lbase + (int64_t)blockIdx.x * lstride;
  double* Wt = wbase + (int64_t)blockIdx.x * b * b;
  extern __shared__ double tsm[];
  double* Wi = tsm;               // 32 x 33 inverse of the diagonal block
  double* Lr = tsm + PNB * PLD;   // 32 x b block row of L (cols < r0)
  __shared__ int bad;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int idx = tid; idx < b * b; idx += blockDim.x) {
    const int r = idx / b, c = idx % b;
    if (c > r) Wt[idx] = 0.0;
  }
  for (int r0 = 0; r0 < b; r0 += PNB) {
    const int nb = min(PNB, b - r0);
    if (tid == 0) bad = -1;
    for (int idx = tid; idx < PNB * PNB; idx += blockDim.x) {
      const int r = idx / PNB, c = idx % PNB;
      Wi[r * PLD + c] = 0.0;
    }
    for (int idx = tid; idx < nb * r0; idx += blockDim.x) {
      const int r = idx / r0, c = idx % r0;
      Lr[r * b + c] = L[(int64_t)(r0 + r) * b + c];
    }
    __syncthreads();
    if (warp == 0) {
      // lane c computes column c of inv(L_rr) by forward substitution
      for (int r = 0; r < nb; ++r) {
        const double d = L[(int64_t)(r0 + r) * b + r0 + r];
        if (d == 0.0 || isnan(d)) {
          if (lane == 0 && bad < 0) bad = r0 + r;
          break;
        }
        if (lane <= r && lane < nb) {
          double acc = (lane == r) ? 1.0 : 0.0;
          for (int k = lane; k < r; ++k)
            acc = fma(-L[(int64_t)(r0 + r) * b + r0 + k], Wi[k * PLD + lane], acc);
          Wi[r * PLD + lane] = acc / d;
        }
        __syncwarp();
      }
    }
    __syncthreads();
    if (bad >= 0) {
      if (tid == 0 && flag) raise_flag(flag, HS_ERR_SINGULAR_BLOCK, column0 + blockIdx.x, bad);
      return;
    }
    for (int idx = tid; idx < nb * nb; idx += blockDim.x) {
      const int r = idx / nb, c = idx % nb;
      if (c <= r) Wt[(int64_t)(r0 + r) * b + r0 + c] = Wi[r * PLD + c];
    }
    // off-diagonal block row
    for (int c = tid; c < r0; c += blockDim.x) {
      double t[PNB];
#pragma unroll
      for (int r = 0; r < PNB; ++r) t[r] = 0.0;
      for (int k = c; k < r0; ++k) {
        const double w = Wt[(int64_t)k * b + c];
#pragma unroll
        for (int r = 0; r < PNB; ++r)
          if (r < nb) t[r] = fma(Lr[r * b + k], w, t[r]);
      }
#pragma unroll
      for (int r = 0; r < PNB; ++r) {
        if (r < nb) {
          double acc = 0.0;
#pragma unroll
          for (int k = 0; k < PNB; ++k)
            if (k <= r) acc = fma(Wi[r * PLD + k], t[k], acc);
          Wt[(int64_t)(r0 + r) * b + c] = -acc;
        }
      }
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// Tile GEMM items. Every mode computes C (+)= -/+ A B^T on b x b tiles whose
// rows are the M / N index and whose columns are the shared K index.

enum GemmMode : int {
  G_UPDATE_ALL = 0,  // column j: A_ik -= X_i X_k^T, j < k <= i
  G_UPDATE_COL = 1,  // column j: only k == j + 1        (lookahead part)
  G_UPDATE_REST = 2, // column j: only k >= j + 2
  G_TRSM = 3,        // column j: X_i = A_ij W_j^T  (out of place)
  G_BATCH = 4,       // C_t -= P_t Q_t^T  (parity tests), lower_only option
};

struct GemmArgs {
  int mode;
  int64_t j;         // column
  int64_t N;         // block rows
  int b;
  int tpd;           // CTA tiles per tile dimension (b / 128)
  double* A;         // packed tiles (local)
  int64_t tile_lo;
  double* X;         // panel workspace: tile i at (i - j - 1) * b*b
  const double* W;   // inverse of L_jj (b*b)
  double* C;         // batch outputs
  const double* P;   // batch A operands
  const double* Q;   // batch B operands
  int lower_only;
  const CholFlag* flag;
};

struct GemmItem {
  const double* a;  // operand tiles (b x b row-major)
  const double* bt;
  double* c;        // output tile
  int64_t a_tile, b_tile;  // tile coordinates for the TMA maps
  int op;           // 0: c -= acc, 1: c = acc
  bool lower;       // write only col <= row (diagonal tiles)
  int kmax;         // K range [0, kmax)
  bool skip;
};

__device__ __forceinline__ GemmItem decode_item(const GemmArgs& g, int64_t item,
                                                int mb, int nb) {
  GemmItem it{};
  const int64_t bb = (int64_t)g.b * g.b;
  it.kmax = g.b;
  if (g.mode == G_TRSM) {
    const int64_t i = g.j + 1 + item;
    it.a = g.A + (tri(i, g.j) - g.tile_lo) * bb;
    it.bt = g.W;
    it.c = g.X + (i - g.j - 1) * bb;
    it.a_tile = tri(i, g.j) - g.tile_lo;
    it.b_tile = 0;
    it.op = 1;
    it.lower = false;
    it.kmax = min(g.b, (nb + 1) * 128);  // W lower: W^T rows > col are zero
    return it;
  }
  if (g.mode == G_BATCH) {
    it.a = g.P + item * bb;
    it.bt = g.Q + item * bb;
    it.c = g.C + item * bb;
    it.a_tile = item;
    it.b_tile = item;
    it.op = 0;
    it.lower = g.lower_only != 0;
    it.skip = it.lower && nb > mb;
    return it;
  }
  int64_t i, k;
  if (g.mode == G_UPDATE_COL) {
    i = g.j + 1 + item;
    k = g.j + 1;
  } else {
    const int64_t base = g.mode == G_UPDATE_REST ? g.j + 2 : g.j + 1;
    const int64_t ii = tile_row(item);
    i = base + ii;
    k = base + (item - tri(ii, 0));
  }
  it.a = g.X + (i - g.j - 1) * bb;
  it.bt = g.X + (k - g.j - 1) * bb;
  it.c = g.A + (tri(i, k) - g.tile_lo) * bb;
  it.a_tile = i - g.j - 1;
  it.b_tile = k - g.j - 1;
  it.op = 0;
  it.lower = (i == k);
  it.skip = it.lower && nb > mb;
  return it;
}

// ---------------------------------------------------------------------------
// DMMA tile GEMM (b % 128 == 0), TMA-fed.

constexpr int GBM = 128, GBN = 128, GKS = 32, GSTAGES = 3;
constexpr int G_OPERAND_BYTES = GBM * GKS * 8;        // 32 KB
constexpr int G_STAGE_BYTES = 2 * G_OPERAND_BYTES;    // A + B
constexpr int G_SMEM = GSTAGES * G_STAGE_BYTES + 1024 + 64;

__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map,
                                            int c0, int c1, int c2,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_"
      "tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void dmma_8x8x4(double (&d)[2], double a, double b) {
  asm volatile(
      "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, "
      "{%0, %1};"
      : "+d"(d[0]), "+d"(d[1])
      : "d"(a), "d"(b));
}

// byte offset of (row, k) inside a [128 rows x 16 k] 128B-swizzled box
__device__ __forceinline__ uint32_t swz(int row, int k) {
  return (uint32_t)(row * 128 + ((((k >> 1) ^ (row & 7))) << 4) + ((k & 1) << 3));
}

__global__ void __launch_bounds__(288, 1)
    gemm_dmma_kernel(const __grid_constant__ CUtensorMap mapA,
                     const __grid_constant__ CUtensorMap mapB, GemmArgs g) {
  if (g.flag && g.flag->status) return;
  const int per = g.tpd * g.tpd;
  const int64_t item = blockIdx.x / per;
  const int sub = (int)(blockIdx.x % per);
  const int mb = sub / g.tpd, nb = sub % g.tpd;
  const GemmItem it = decode_item(g, item, mb, nb);
  if (it.skip) return;
  const int nks = it.kmax / GKS;

  extern __shared__ __align__(1024) unsigned char gsm_raw[];
  unsigned char* gsm = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(gsm_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(gsm + GSTAGES * G_STAGE_BYTES);
  uint64_t* empty = full + GSTAGES;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int s = 0; s < GSTAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 8);
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (warp == 8) {
    if (lane == 0) {
      const int arow = mb * GBM, brow = nb * GBN;
      for (int ks = 0; ks < nks; ++ks) {
        const int st = ks % GSTAGES;
        if (ks >= GSTAGES) mbar_wait(&empty[st], ((ks / GSTAGES) - 1) & 1);
        unsigned char* sa = gsm + st * G_STAGE_BYTES;
        unsigned char* sb = sa + G_OPERAND_BYTES;
        mbar_arrive_expect_tx(&full[st], G_STAGE_BYTES);
        const int k0 = ks * GKS;
        tma_load_3d(sa, &mapA, k0, arow, (int)it.a_tile, &full[st]);
        tma_load_3d(sa + G_OPERAND_BYTES / 2, &mapA, k0 + 16, arow,
                    (int)it.a_tile, &full[st]);
        tma_load_3d(sb, &mapB, k0, brow, (int)it.b_tile, &full[st]);
        tma_load_3d(sb + G_OPERAND_BYTES / 2, &mapB, k0 + 16, brow,
                    (int)it.b_tile, &full[st]);
      }
    }
    return;
  }

  const int wm = warp & 3, wn = warp >> 2;  // 4 x 2 warps of 32 x 64
  double acc[4][8][2];
#pragma unroll
  for (int x = 0; x < 4; ++x)
#pragma unroll
    for (int y = 0; y < 8; ++y) acc[x][y][0] = acc[x][y][1] = 0.0;
  const int fr = lane >> 2, fk = lane & 3;

  for (int ks = 0; ks < nks; ++ks) {
    const int st = ks % GSTAGES;
    mbar_wait(&full[st], (ks / GSTAGES) & 1);
    const unsigned char* sa = gsm + st * G_STAGE_BYTES;
    const unsigned char* sb = sa + G_OPERAND_BYTES;
#pragma unroll
    for (int kk = 0; kk < GKS / 4; ++kk) {
      const int k = kk * 4 + fk;  // 0..31
      const unsigned char* ba = sa + (k >> 4) * (G_OPERAND_BYTES / 2);
      const unsigned char* bbp = sb + (k >> 4) * (G_OPERAND_BYTES / 2);
      double af[4], bf[8];
#pragma unroll
      for (int x = 0; x < 4; ++x)
        af[x] = *reinterpret_cast<const double*>(ba + swz(wm * 32 + x * 8 + fr, k & 15));
#pragma unroll
      for (int y = 0; y < 8; ++y)
        bf[y] = *reinterpret_cast<const double*>(bbp + swz(wn * 64 + y * 8 + fr, k & 15));
#pragma unroll
      for (int x = 0; x < 4; ++x)
#pragma unroll
        for (int y = 0; y < 8; ++y) dmma_8x8x4(acc[x][y], af[x], bf[y]);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[st]);
  }

  // epilogue: C rows (mb*128 + wm*32 + x*8 + fr), cols (nb*128 + wn*64 +
  // y*8 + 2*fk + {0,1})
  const int b = g.b;
#pragma unroll
  for (int x = 0; x < 4; ++x) {
    const int row = mb * GBM + wm * 32 + x * 8 + fr;
#pragma unroll
    for (int y = 0; y < 8; ++y) {
      const int col = nb * GBN + wn * 64 + y * 8 + 2 * fk;
      double2* p = reinterpret_cast<double2*>(it.c + (int64_t)row * b + col);
      if (it.op == 1) {
        *p = make_double2(acc[x][y][0], acc[x][y][1]);
      } else if (!it.lower || col + 1 <= row) {
        double2 v = *p;
        v.x -= acc[x][y][0];
        v.y -= acc[x][y][1];
        *p = v;
      } else if (col <= row) {
        it.c[(int64_t)row * b + col] -= acc[x][y][0];
      }
    }
  }
}

// ---------------------------------------------------------------------------
// SIMT FP64 tile GEMM (any b): 64 x 64 CTA tile, 4 x 4 per thread, K chunks
// of 16 staged in shared memory.

__global__ void __launch_bounds__(256) gemm_simt_kernel(GemmArgs g) {
  if (g.flag && g.flag->status) return;
  const int b = g.b;
  const int tpd = (b + 63) / 64;
  const int per = tpd * tpd;
  const int64_t item = blockIdx.x / per;
  const int sub = (int)(blockIdx.x % per);
  const int mb = sub / tpd, nb = sub % tpd;
  GemmItem it = decode_item(g, item, mb, nb);
  // recompute skip / kmax at 64 granularity
  if (it.lower && nb > mb) return;
  if (g.mode == G_TRSM) it.kmax = min(b, (nb + 1) * 64);
  __shared__ double As[16][65], Bs[16][65];
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  double acc[4][4];
#pragma unroll
  for (int x = 0; x < 4; ++x)
#pragma unroll
    for (int y = 0; y < 4; ++y) acc[x][y] = 0.0;
  const int m0 = mb * 64, n0 = nb * 64;
  for (int k0 = 0; k0 < it.kmax; k0 += 16) {
    for (int idx = threadIdx.x; idx < 64 * 16; idx += 256) {
      const int r = idx / 16, k = idx % 16;
      const int gr = m0 + r, gn = n0 + r, gk = k0 + k;
      As[k][r] = (gr < b && gk < it.kmax) ? it.a[(int64_t)gr * b + gk] : 0.0;
      Bs[k][r] = (gn < b && gk < it.kmax) ? it.bt[(int64_t)gn * b + gk] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      double a[4], bq[4];
#pragma unroll
      for (int x = 0; x < 4; ++x) a[x] = As[k][ty * 4 + x];
#pragma unroll
      for (int y = 0; y < 4; ++y) bq[y] = Bs[k][tx * 4 + y];
#pragma unroll
      for (int x = 0; x < 4; ++x)
#pragma unroll
        for (int y = 0; y < 4; ++y) acc[x][y] = fma(a[x], bq[y], acc[x][y]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int x = 0; x < 4; ++x)
#pragma unroll
    for (int y = 0; y < 4; ++y) {
      const int row = m0 + ty * 4 + x, col = n0 + tx * 4 + y;
      if (row >= b || col >= b) continue;
      if (it.lower && col > row) continue;
      double* p = it.c + (int64_t)row * b + col;
      if (it.op == 1) *p = acc[x][y];
      else *p -= acc[x][y];
    }
}

// ---------------------------------------------------------------------------
// small kernels

// A_ij <- X_i for i in (j, N)
__global__ void copy_panel_kernel(double* A, int64_t tile_lo, const double* X,
                                  int64_t j, int b, const CholFlag* flag) {
  if (flag->status) return;
  const int64_t i = j + 1 + blockIdx.y;
  const int64_t bb = (int64_t)b * b;
  const double* src = X + (i - j - 1) * bb;
  double* dst = A + (tri(i, j) - tile_lo) * bb;
  if ((bb & 1) == 0) {
    const double2* s2 = reinterpret_cast<const double2*>(src);
    double2* d2 = reinterpret_cast<double2*>(dst);
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < bb / 2;
         k += (int64_t)gridDim.x * blockDim.x)
      d2[k] = s2[k];
  } else {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < bb;
         k += (int64_t)gridDim.x * blockDim.x)
      dst[k] = src[k];
  }
}

// NaN/Inf scan of the lower triangles (cholesky_solver.cpp:222-238)
__global__ void check_finite_kernel(const double* A, int64_t tile_lo,
                                    int64_t ntiles, int b, CholFlag* flag) {
  const int64_t bb = (int64_t)b * b;
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int64_t gt = tile_lo + t;
    const int64_t i = tile_row(gt), j = gt - tri(i, 0);
    const double* blk = A + t * bb;
    for (int idx = threadIdx.x; idx < bb; idx += blockDim.x) {
      const int r = idx / b, c = idx % b;
      if (i == j && c > r) continue;
      if (!isfinite(blk[idx])) raise_flag(flag, HS_ERR_NUMERICAL, i, j);
    }
  }
}

// ---- triangular solves with the stored inverses ---------------------------
// forward row i: s = v_i - sum_{j<i} L_ij v_j ; v_i = W_i s
// back row i:    s = v_i - sum_{j>i} L_ji^T v_j ; v_i = W_i^T s
// Stage 1: CTA (tile jj, 32-row/col chunk) writes a partial; stage 2 sums
// partials in fixed order and applies the inverse.

__global__ void trsv_partial_kernel(const double* A, int64_t tile_lo,
                                    const double* v, int b, int64_t i,
                                    int upper, double* part,
                                    const CholFlag* flag) {
  if (flag && flag->status) return;
  const int64_t jj = blockIdx.y;  // j index among the contributing tiles
  const int chunk = blockIdx.x;   // 32 outputs
  const int64_t bb = (int64_t)b * b;
  __shared__ double vs[1024];
  __shared__ double red[8][33];
  int64_t tile, vj;
  if (!upper) {
    tile = tri(i, jj);
    vj = jj;
  } else {
    tile = tri(i + 1 + jj, i);
    vj = i + 1 + jj;
  }
  const double* T = A + (tile - tile_lo) * bb;
  for (int k = threadIdx.x; k < b; k += blockDim.x) vs[k] = v[vj * b + k];
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int o0 = chunk * 32;
  if (!upper) {
    // outputs r in [o0, o0+32): sum_c T[r][c] vs[c]; warp w takes rows
    for (int rr = warp; rr < 32; rr += 8) {
      const int r = o0 + rr;
      double acc = 0.0;
      if (r < b)
        for (int c = lane; c < b; c += 32) acc = fma(T[(int64_t)r * b + c], vs[c], acc);
      for (int off = 16; off; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
      if (lane == 0 && r < b) part[jj * b + r] = acc;
    }
  } else {
    // outputs c in [o0, o0+32): sum_r T[r][c] vs[r]; lane = column
    const int c = o0 + lane;
    double acc = 0.0;
    if (c < b)
      for (int r = warp; r < b; r += 8) acc = fma(T[(int64_t)r * b + c], vs[r], acc);
    red[warp][lane] = acc;
    __syncthreads();
    if (warp == 0 && c < b) {
      double s = 0.0;
      for (int w = 0; w < 8; ++w) s += red[w][lane];
      part[jj * b + c] = s;
    }
  }
}

__global__ void trsv_apply_kernel(const double* W, const double* rhs, double* v,
                                  int b, int64_t i, int upper,
                                  const double* part, int64_t nparts,
                                  const CholFlag* flag) {
  if (flag && flag->status) return;
  __shared__ double s[1024];
  for (int k = threadIdx.x; k < b; k += blockDim.x) {
    double acc = rhs[i * b + k];
    for (int64_t p = 0; p < nparts; ++p) acc -= part[p * b + k];
    s[k] = acc;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nw = blockDim.x >> 5;
  const int o0 = blockIdx.x * 32;
  if (!upper) {
    for (int rr = warp; rr < 32; rr += nw) {
      const int r = o0 + rr;
      if (r >= b) break;
      double acc = 0.0;
      for (int c = lane; c <= r; c += 32) acc = fma(W[(int64_t)r * b + c], s[c], acc);
      for (int off = 16; off; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
      if (lane == 0) v[i * b + r] = acc;
    }
  } else {
    // (W^T s)[c] = sum_{r >= c} W[r][c] s[r]
    __shared__ double red[32][33];
    const int c = o0 + lane;
    double acc = 0.0;
    if (c < b)
      for (int r = c + warp; r < b; r += nw) acc = fma(W[(int64_t)r * b + c], s[r], acc);
    red[warp][lane] = acc;
    __syncthreads();
    if (warp == 0 && c < b) {
      double t = 0.0;
      for (int w = 0; w < nw; ++w) t += red[w][lane];
      v[i * b + c] = t;
    }
  }
}

// ---------------------------------------------------------------------------
// host side

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t,
                                  void*, const cuuint64_t*, const cuuint64_t*,
                                  const cuuint32_t*, const cuuint32_t*,
                                  CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion,
                                  CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    HS_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p,
                                    cudaEnableDefault, &q));
    HS_REQUIRE(p && q == cudaDriverEntryPointSuccess, HS_ERR_CUDA,
               "cuTensorMapEncodeTiled unavailable");
    fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

// 3-D map over `ntiles` contiguous b x b tiles: box 16 (k) x 128 (rows) x 1.
static CUtensorMap tile_map(const double* base, int b, int64_t ntiles) {
  CUtensorMap m;
  cuuint64_t dims[3] = {(cuuint64_t)b, (cuuint64_t)b,
                        (cuuint64_t)std::max<int64_t>(ntiles, 1)};
  cuuint64_t strides[2] = {(cuuint64_t)b * 8, (cuuint64_t)b * b * 8};
  cuuint32_t box[3] = {16, 128, 1};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3,
                           const_cast<double*>(base), dims, strides, box, es,
                           CU_TENSOR_MAP_INTERLEAVE_NONE,
                           CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  HS_REQUIRE(r == CUDA_SUCCESS, HS_ERR_CUDA, "cuTensorMapEncodeTiled failed");
  return m;
}

static bool dmma_ok(int b) { return b % 128 == 0; }

static void launch_gemm(hs_ctx* c, cudaStream_t s, const GemmArgs& g,
                        int64_t items, const CUtensorMap* ma,
                        const CUtensorMap* mb) {
  if (items <= 0) return;
  if (dmma_ok(g.b) && ma && mb) {
    static bool attr = false;
    if (!attr) {
      HS_CUDA(cudaFuncSetAttribute(gemm_dmma_kernel,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   G_SMEM));
      attr = true;
    }
    const int64_t grid = items * g.tpd * g.tpd;
    gemm_dmma_kernel<<<(unsigned)grid, 288, G_SMEM, s>>>(*ma, *mb, g);
  } else {
    const int tpd = (g.b + 63) / 64;
    const int64_t grid = items * tpd * tpd;
    gemm_simt_kernel<<<(unsigned)grid, 256, 0, s>>>(g);
  }
  HS_CUDA(cudaGetLastError());
  launch_count(c);
}

static size_t potrf_smem(int b) { return (size_t)(PNB * PLD + b * PLD) * 8; }
static size_t trtri_smem(int b) { return (size_t)(PNB * PLD + PNB * b) * 8; }

static void set_tile_kernel_attrs(int b) {
  HS_REQUIRE(potrf_smem(b) <= 227 * 1024 && trtri_smem(b) <= 227 * 1024,
             HS_ERR_CONFIG, "block size too large for the tile kernels (max 768)");
  HS_CUDA(cudaFuncSetAttribute(potrf_tile_kernel,
                               cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)potrf_smem(b)));
  HS_CUDA(cudaFuncSetAttribute(trtri_tile_kernel,
                               cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)trtri_smem(b)));
}

struct ColStreams {
  cudaStream_t p = nullptr, u = nullptr;
  std::vector<cudaEvent_t> ev;
  ~ColStreams() {
    for (auto e : ev) cudaEventDestroy(e);
    if (p) cudaStreamDestroy(p);
    if (u) cudaStreamDestroy(u);
  }
  cudaEvent_t make() {
    cudaEvent_t e;
    HS_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    ev.push_back(e);
    return e;
  }
};

static double ms_since(std::chrono::steady_clock::time_point t0) {
  return std::chrono::duration<double, std::milli>(
             std::chrono::steady_clock::now() - t0)
      .count();
}

// In-place factorization of a single-rank matrix.
static void potrf_run(hs_ctx* c, hs_matrix* m) {
  HS_REQUIRE(c->world == 1, HS_ERR_CONFIG,
             "multi-GPU Cholesky is not available in this build");
  const int b = (int)m->b;
  const int64_t N = (int64_t)m->N;
  const int64_t bb = (int64_t)b * b;
  set_tile_kernel_attrs(b);
  if (!m->dinv) HS_CUDA(cudaMalloc(&m->dinv, N * bb * sizeof(double)));
  m->has_inv = false;
  CholFlag* flag = nullptr;
  double* X[2] = {nullptr, nullptr};
  HS_CUDA(cudaMalloc(&flag, sizeof(CholFlag)));
  struct Guard {
    CholFlag* f;
    double** x;
    ~Guard() {
      cudaFree(f);
      cudaFree(x[0]);
      cudaFree(x[1]);
    }
  } guard{flag, X};
  const int64_t panel = std::max<int64_t>(N - 1, 1);
  HS_CUDA(cudaMalloc(&X[0], panel * bb * sizeof(double)));
  HS_CUDA(cudaMalloc(&X[1], panel * bb * sizeof(double)));
  HS_CUDA(cudaMemsetAsync(flag, 0, sizeof(CholFlag), c->stream));

  ColStreams cs;
  int lo_pri, hi_pri;
  HS_CUDA(cudaDeviceGetStreamPriorityRange(&lo_pri, &hi_pri));
  HS_CUDA(cudaStreamCreateWithPriority(&cs.p, cudaStreamNonBlocking, hi_pri));
  HS_CUDA(cudaStreamCreateWithPriority(&cs.u, cudaStreamNonBlocking, lo_pri));
  cudaEvent_t start = cs.make();
  HS_CUDA(cudaEventRecord(start, c->stream));
  HS_CUDA(cudaStreamWaitEvent(cs.p, start));
  HS_CUDA(cudaStreamWaitEvent(cs.u, start));

  const bool fast = dmma_ok(b);
  CUtensorMap mapA{}, mapX[2]{};
  if (fast) {
    mapA = tile_map(m->d, b, (int64_t)m->local_tiles());
    mapX[0] = tile_map(X[0], b, panel);
    mapX[1] = tile_map(X[1], b, panel);
  }

  GemmArgs g{};
  g.N = N;
  g.b = b;
  g.tpd = b / 128;
  g.A = m->d;
  g.tile_lo = m->tile_lo;
  g.flag = flag;

  // P-stream work for column j: potrf, trtri, trsm into X[j&1], copy back.
  auto panel_work = [&](int64_t j) {
    double* djj = m->d + (tri(j, j) - m->tile_lo) * bb;
    double* wj = m->dinv + j * bb;
    potrf_tile_kernel<<<1, 256, potrf_smem(b), cs.p>>>(djj, 0, b, flag, j);
    HS_CUDA(cudaGetLastError());
    trtri_tile_kernel<<<1, 256, trtri_smem(b), cs.p>>>(djj, 0, wj, b, flag, j);
    HS_CUDA(cudaGetLastError());
    launch_count(c, 2);
    const int64_t t = N - 1 - j;
    if (t > 0) {
      GemmArgs gt = g;
      gt.mode = G_TRSM;
      gt.j = j;
      gt.X = X[j & 1];
      gt.W = wj;
      CUtensorMap mw;
      if (fast) mw = tile_map(wj, b, 1);
      launch_gemm(c, cs.p, gt, t, fast ? &mapA : nullptr, fast ? &mw : nullptr);
      dim3 grid((unsigned)std::max<int64_t>(1, std::min<int64_t>(64, ceil_div(bb, 512))),
                (unsigned)t);
      copy_panel_kernel<<<grid, 256, 0, cs.p>>>(m->d, m->tile_lo, X[j & 1], j, b,
                                                flag);
      HS_CUDA(cudaGetLastError());
      launch_count(c);
    }
  };

  panel_work(0);
  for (int64_t j = 0; j < N; ++j) {
    const int64_t t = N - 1 - j;
    cudaEvent_t pdone = cs.make();
    HS_CUDA(cudaEventRecord(pdone, cs.p));
    if (t == 0) break;
    HS_CUDA(cudaStreamWaitEvent(cs.u, pdone));
    GemmArgs gu = g;
    gu.j = j;
    gu.X = X[j & 1];
    const CUtensorMap* mx = fast ? &mapX[j & 1] : nullptr;
    // lookahead: tile column j+1 first
    gu.mode = G_UPDATE_COL;
    launch_gemm(c, cs.u, gu, t, mx, mx);
    cudaEvent_t ucol = cs.make();
    HS_CUDA(cudaEventRecord(ucol, cs.u));
    HS_CUDA(cudaStreamWaitEvent(cs.p, ucol));
    // the rest of column j's update overlaps column j+1's panel work; the
    // panel writes X[(j+1)&1], the update reads X[j&1]
    gu.mode = G_UPDATE_REST;
    const int64_t tr = t - 1;
    launch_gemm(c, cs.u, gu, tr * (tr + 1) / 2, mx, mx);
    // X[(j+1)&1] is about to be overwritten: the update of column j-1 (which
    // read it) is ordered before this point on cs.u, and P waited on ucol.
    panel_work(j + 1);
  }
  cudaEvent_t pend = cs.make(), uend = cs.make();
  HS_CUDA(cudaEventRecord(pend, cs.p));
  HS_CUDA(cudaEventRecord(uend, cs.u));
  HS_CUDA(cudaStreamWaitEvent(c->stream, pend));
  HS_CUDA(cudaStreamWaitEvent(c->stream, uend));
  // check_finite (only when no earlier failure)
  check_finite_kernel<<<(unsigned)std::min<int64_t>(m->local_tiles(), 4 * 148), 256,
                        0, c->stream>>>(m->d, m->tile_lo, (int64_t)m->local_tiles(),
                                        b, flag);
  HS_CUDA(cudaGetLastError());
  launch_count(c);
  CholFlag h{};
  HS_CUDA(cudaMemcpyAsync(&h, flag, sizeof(h), cudaMemcpyDeviceToHost, c->stream));
  HS_CUDA(cudaStreamSynchronize(c->stream));
  if (h.status == HS_ERR_NOT_SPD)
    throw Failure{HS_ERR_NOT_SPD,
                  "matrix is not positive definite (block row " +
                      std::to_string(h.col) + ", pivot " + std::to_string(h.pivot) + ")",
                  h.col, h.pivot};
  if (h.status == HS_ERR_NUMERICAL)
    throw Failure{HS_ERR_NUMERICAL,
                  "factor has a non-finite value in block (" + std::to_string(h.col) +
                      ", " + std::to_string(h.pivot) + ")",
                  h.col, h.pivot};
  if (h.status != HS_OK)
    throw Failure{h.status, "factorization failed", h.col, h.pivot};
  m->has_inv = true;
}

// inverses of all diagonal tiles of an (uploaded) factor; singular check
static void ensure_inverses(hs_ctx* c, hs_matrix* m) {
  if (m->has_inv) return;
  const int b = (int)m->b;
  const int64_t N = (int64_t)m->N;
  const int64_t bb = (int64_t)b * b;
  set_tile_kernel_attrs(b);
  if (!m->dinv) HS_CUDA(cudaMalloc(&m->dinv, N * bb * sizeof(double)));
  CholFlag* flag = nullptr;
  HS_CUDA(cudaMalloc(&flag, sizeof(CholFlag)));
  HS_CUDA(cudaMemsetAsync(flag, 0, sizeof(CholFlag), c->stream));
  // diagonal tile j sits at tri(j, j); launch one CTA per tile row j
  for (int64_t j = 0; j < N; ++j) {
    trtri_tile_kernel<<<1, 256, trtri_smem(b), c->stream>>>(
        m->d + (tri(j, j) - m->tile_lo) * bb, 0, m->dinv + j * bb, b, flag, j);
    HS_CUDA(cudaGetLastError());
  }
  launch_count(c, (int)N);
  CholFlag h{};
  HS_CUDA(cudaMemcpyAsync(&h, flag, sizeof(h), cudaMemcpyDeviceToHost, c->stream));
  HS_CUDA(cudaStreamSynchronize(c->stream));
  cudaFree(flag);
  if (h.status == HS_ERR_SINGULAR_BLOCK)
    throw Failure{HS_ERR_SINGULAR_BLOCK,
                  "triangular block has zero or NaN diagonal at index " +
                      std::to_string(h.pivot),
                  h.col, h.pivot};
  m->has_inv = true;
}

static void trsv_run(hs_ctx* c, hs_matrix* m, double* v, bool upper) {
  HS_REQUIRE(c->world == 1, HS_ERR_CONFIG, "triangular solves are single-rank");
  ensure_inverses(c, m);
  const int b = (int)m->b;
  HS_REQUIRE(b <= 1024, HS_ERR_CONFIG, "block size > 1024 unsupported in trsv");
  const int64_t N = (int64_t)m->N;
  const int64_t bb = (int64_t)b * b;
  // rhs snapshot: the apply step reads row i of it and writes row i of v,
  // so CTAs of one row never read values another CTA already overwrote
  double *part = nullptr, *rhs = nullptr;
  HS_CUDA(cudaMalloc(&part, std::max<int64_t>(N, 1) * b * sizeof(double)));
  HS_CUDA(cudaMalloc(&rhs, N * b * sizeof(double)));
  HS_CUDA(cudaMemcpyAsync(rhs, v, N * b * sizeof(double),
                          cudaMemcpyDeviceToDevice, c->stream));
  const int chunks = (b + 31) / 32;
  for (int64_t s = 0; s < N; ++s) {
    const int64_t i = upper ? N - 1 - s : s;
    const int64_t np = upper ? N - 1 - i : i;
    if (np > 0) {
      trsv_partial_kernel<<<dim3(chunks, (unsigned)np), 256, 0, c->stream>>>(
          m->d, m->tile_lo, v, b, i, upper ? 1 : 0, part, nullptr);
      HS_CUDA(cudaGetLastError());
      launch_count(c);
    }
    trsv_apply_kernel<<<chunks, 256, 0, c->stream>>>(m->dinv + i * bb, rhs, v,
                                                     b, i, upper ? 1 : 0, part,
                                                     np, nullptr);
    HS_CUDA(cudaGetLastError());
    launch_count(c);
  }
  HS_CUDA(cudaStreamSynchronize(c->stream));
  cudaFree(part);
  cudaFree(rhs);
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

hs_status hs_potrf(hs_ctx* c, hs_matrix* m, hs_chol_stats* st) {
  HS_API_BEGIN
  HS_REQUIRE(c && m, HS_ERR_CONFIG, "null pointer");
  HS_CUDA(cudaSetDevice(c->device));
  const auto t0 = std::chrono::steady_clock::now();
  potrf_run(c, m);
  if (st) {
    std::memset(st, 0, sizeof(*st));
    st->factor_ms = ms_since(t0);
    st->wall_ms = st->compute_ms = st->factor_ms;
  }
  HS_API_END
}

hs_status hs_trsv_lower(hs_ctx* c, const hs_matrix* l, double* d_v) {
  HS_API_BEGIN
  HS_REQUIRE(c && l && d_v, HS_ERR_CONFIG, "null pointer");
  HS_CUDA(cudaSetDevice(c->device));
  trsv_run(c, const_cast<hs_matrix*>(l), d_v, false);
  HS_API_END
}

hs_status hs_trsv_upper(hs_ctx* c, const hs_matrix* l, double* d_v) {
  HS_API_BEGIN
  HS_REQUIRE(c && l && d_v, HS_ERR_CONFIG, "null pointer");
  HS_CUDA(cudaSetDevice(c->device));
  trsv_run(c, const_cast<hs_matrix*>(l), d_v, true);
  HS_API_END
}

hs_status hs_solve_spd(hs_ctx* c, hs_matrix* a, const double* d_rhs,
                       double* d_x, const hs_matrix* a_orig,
                       hs_chol_stats* st) {
  HS_API_BEGIN
  HS_REQUIRE(c && a && d_rhs && d_x, HS_ERR_CONFIG, "null pointer");
  HS_CUDA(cudaSetDevice(c->device));
  hs_chol_stats s{};
  const auto t0 = std::chrono::steady_clock::now();
  potrf_run(c, a);
  s.factor_ms = ms_since(t0);
  const auto t1 = std::chrono::steady_clock::now();
  const size_t pn = a->N * a->b;
  HS_CUDA(cudaMemcpyAsync(d_x, d_rhs, pn * sizeof(double),
                          cudaMemcpyDeviceToDevice, c->stream));
  trsv_run(c, a, d_x, false);
  trsv_run(c, a, d_x, true);
  s.solve_ms = ms_since(t1);
  s.wall_ms = ms_since(t0);
  s.compute_ms = s.wall_ms;
  if (a_orig) {
    hs_status r = hs_true_residual(c, a_orig, d_x, d_rhs, &s.true_residual);
    if (r != HS_OK) throw Failure{r, hs_last_error()};
  }
  if (st) *st = s;
  HS_API_END
}

hs_status hs_factorize_host(hs_ctx* c, size_t n, size_t b, double* a_packed,
                            hs_chol_stats* st) {
  HS_API_BEGIN
  HS_REQUIRE(c && a_packed, HS_ERR_CONFIG, "null pointer");
  HS_CUDA(cudaSetDevice(c->device));
  hs_matrix* m = nullptr;
  hs_status s = hs_matrix_create(c, n, b, &m);
  if (s != HS_OK) throw Failure{s, hs_last_error()};
  struct G {
    hs_matrix* m;
    ~G() { hs_matrix_destroy(m); }
  } guard{m};
  const auto t0 = std::chrono::steady_clock::now();
  s = hs_matrix_upload(m, a_packed);
  if (s != HS_OK) throw Failure{s, hs_last_error()};
  const double up = ms_since(t0);
  const auto t1 = std::chrono::steady_clock::now();
  potrf_run(c, m);
  const double fac = ms_since(t1);
  const auto t2 = std::chrono::steady_clock::now();
  s = hs_matrix_download(m, a_packed);
  if (s != HS_OK) throw Failure{s, hs_last_error()};
  if (st) {
    std::memset(st, 0, sizeof(*st));
    st->factor_ms = ms_since(t0);
    st->transfer_ms = up + ms_since(t2);
    st->compute_ms = fac;
    st->wall_ms = st->factor_ms;
  }
  HS_API_END
}

hs_status hs_solve_spd_host(hs_ctx* c, size_t n, size_t b, double* a_packed,
                            const double* rhs, double* x, hs_chol_stats* st) {
  HS_API_BEGIN
  HS_REQUIRE(c && a_packed && rhs && x, HS_ERR_CONFIG, "null pointer");
  HS_CUDA(cudaSetDevice(c->device));
  hs_matrix *m = nullptr, *orig = nullptr;
  hs_status s = hs_matrix_create(c, n, b, &m);
  if (s != HS_OK) throw Failure{s, hs_last_error()};
  s = hs_matrix_create(c, n, b, &orig);
  if (s != HS_OK) {
    hs_matrix_destroy(m);
    throw Failure{s, hs_last_error()};
  }
  double *d_rhs = nullptr, *d_x = nullptr;
  struct G {
    hs_matrix *a, *b;
    double **r, **x;
    ~G() {
      hs_matrix_destroy(a);
      hs_matrix_destroy(b);
      cudaFree(*r);
      cudaFree(*x);
    }
  } guard{m, orig, &d_rhs, &d_x};
  const size_t pn = (size_t)ceil_div(n, b) * b;
  HS_CUDA(cudaMalloc(&d_rhs, pn * sizeof(double)));
  HS_CUDA(cudaMalloc(&d_x, pn * sizeof(double)));
  const auto t0 = std::chrono::steady_clock::now();
  s = hs_matrix_upload(m, a_packed);
  if (s != HS_OK) throw Failure{s, hs_last_error()};
  HS_CUDA(cudaMemcpyAsync(d_rhs, rhs, pn * sizeof(double), cudaMemcpyHostToDevice,
                          c->stream));
  HS_CUDA(cudaMemcpyAsync(orig->d, m->d, m->local_tiles() * b * b * sizeof(double),
                          cudaMemcpyDeviceToDevice, c->stream));
  HS_CUDA(cudaStreamSynchronize(c->stream));
  const double up = ms_since(t0);
  hs_chol_stats in{};
  s = hs_solve_spd(c, m, d_rhs, d_x, orig, &in);
  if (s != HS_OK) throw Failure{s, hs_last_error(), -1, -1};
  const auto t2 = std::chrono::steady_clock::now();
  HS_CUDA(cudaMemcpyAsync(x, d_x, pn * sizeof(double), cudaMemcpyDeviceToHost,
                          c->stream));
  s = hs_matrix_download(m, a_packed);
  if (s != HS_OK) throw Failure{s, hs_last_error()};
  if (st) {
    *st = in;
    st->transfer_ms = up + ms_since(t2);
    st->wall_ms = ms_since(t0);
  }
  HS_API_END
}

hs_status hs_forward_substitute_host(hs_ctx* c, size_t n, size_t b,
                                     const double* l, const double* rhs,
                                     double* y) {
  HS_API_BEGIN
  HS_REQUIRE(c && l && rhs && y, HS_ERR_CONFIG, "null pointer");
  HS_CUDA(cudaSetDevice(c->device));
  hs_matrix* m = nullptr;
  hs_status s = hs_matrix_create(c, n, b, &m);
  if (s != HS_OK) throw Failure{s, hs_last_error()};
  double* d_v = nullptr;
  struct G {
    hs_matrix* m;
    double** v;
    ~G() {
      hs_matrix_destroy(m);
      cudaFree(*v);
    }
  } guard{m, &d_v};
  s = hs_matrix_upload(m, l);
  if (s != HS_OK) throw Failure{s, hs_last_error()};
  const size_t pn = (size_t)ceil_div(n, b) * b;
  HS_CUDA(cudaMalloc(&d_v, pn * sizeof(double)));
  HS_CUDA(cudaMemcpy(d_v, rhs, pn * sizeof(double), cudaMemcpyHostToDevice));
  trsv_run(c, m, d_v, false);
  HS_CUDA(cudaMemcpy(y, d_v, pn * sizeof(double), cudaMemcpyDeviceToHost));
  HS_API_END
}

hs_status hs_back_substitute_host(hs_ctx* c, size_t n, size_t b,
                                  const double* l, const double* yv,
                                  double* x) {
  HS_API_BEGIN
  HS_REQUIRE(c && l && yv && x, HS_ERR_CONFIG, "null pointer");
  HS_CUDA(cudaSetDevice(c->device));
  hs_matrix* m = nullptr;
  hs_status s = hs_matrix_create(c, n, b, &m);
  if (s != HS_OK) throw Failure{s, hs_last_error()};
  double* d_v = nullptr;
  struct G {
    hs_matrix* m;
    double** v;
    ~G() {
      hs_matrix_destroy(m);
      cudaFree(*v);
    }
  } guard{m, &d_v};
  s = hs_matrix_upload(m, l);
  if (s != HS_OK) throw Failure{s, hs_last_error()};
  const size_t pn = (size_t)ceil_div(n, b) * b;
  HS_CUDA(cudaMalloc(&d_v, pn * sizeof(double)));
  HS_CUDA(cudaMemcpy(d_v, yv, pn * sizeof(double), cudaMemcpyHostToDevice));
  trsv_run(c, m, d_v, true);
  HS_CUDA(cudaMemcpy(x, d_v, pn * sizeof(double), cudaMemcpyDeviceToHost));
  HS_API_END
}

hs_status hs_potf_tiles(hs_ctx* c, double* d_tiles, size_t b, size_t count,
                        int64_t* first_bad_pivot) {
  HS_API_BEGIN
  HS_REQUIRE(c && d_tiles && b > 0, HS_ERR_CONFIG, "bad arguments");
  HS_CUDA(cudaSetDevice(c->device));
  set_tile_kernel_attrs((int)b);
  CholFlag* flag = nullptr;
  HS_CUDA(cudaMalloc(&flag, sizeof(CholFlag)));
  HS_CUDA(cudaMemsetAsync(flag, 0, sizeof(CholFlag), c->stream));
  potrf_tile_kernel<<<(unsigned)count, 256, potrf_smem((int)b), c->stream>>>(
      d_tiles, (int64_t)(b * b), (int)b, flag, -1);
  HS_CUDA(cudaGetLastError());
  launch_count(c);
  CholFlag h{};
  HS_CUDA(cudaMemcpyAsync(&h, flag, sizeof(h), cudaMemcpyDeviceToHost, c->stream));
  HS_CUDA(cudaStreamSynchronize(c->stream));
  cudaFree(flag);
  if (first_bad_pivot) *first_bad_pivot = h.status ? h.pivot : -1;
  if (h.status)
    throw Failure{h.status,
                  "matrix is not positive definite (block row -1, pivot " +
                      std::to_string(h.pivot) + ")",
                  -1, h.pivot};
  HS_API_END
}

hs_status hs_gemm_update_tiles(hs_ctx* c, double* d_c, const double* d_p,
                               const double* d_q, size_t b, size_t count,
                               int lower_only) {
  HS_API_BEGIN
  HS_REQUIRE(c && d_c && d_p && d_q && b > 0, HS_ERR_CONFIG, "bad arguments");
  HS_CUDA(cudaSetDevice(c->device));
  GemmArgs g{};
  g.mode = G_BATCH;
  g.b = (int)b;
  g.tpd = (int)b / 128;
  g.C = d_c;
  g.P = d_p;
  g.Q = d_q;
  g.lower_only = lower_only;
  if (dmma_ok((int)b)) {
    CUtensorMap mp = tile_map(d_p, (int)b, (int64_t)count);
    CUtensorMap mq = tile_map(d_q, (int)b, (int64_t)count);
    launch_gemm(c, c->stream, g, (int64_t)count, &mp, &mq);
  } else {
    launch_gemm(c, c->stream, g, (int64_t)count, nullptr, nullptr);
  }
  HS_CUDA(cudaStreamSynchronize(c->stream));
  HS_API_END
}

}  // extern "C"
