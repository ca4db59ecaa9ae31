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
    trtri_tile_kernel(const double* A, int64_t tile_lo, double* wbase, int b,
                      CholFlag* flag, int64_t j0) {
  if (flag && flag->status) return;
  const int64_t jt = j0 + blockIdx.x;  // diagonal tile (jt, jt)
  const double* L = A + (tri(jt, jt) - tile_lo) * b * b;
  double* Wt = wbase + jt * b * b;
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
      if (tid == 0 && flag) raise_flag(flag, HS_ERR_SINGULAR_BLOCK, jt, bad);
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
// Sub-block GEMM. Every item computes one cb x cb output sub-block
//   C  =  A_op B_op^T          (op SET)   or
//   C -=  A_op B_op^T          (op SUB, lower-only on diagonal sub-blocks)
// where A_op / B_op are cb x K row strips of packed tiles (k contiguous) or
// of the inverse blocks. cb = 128 on the DMMA path (b % 128 == 0); on the
// SIMT path cb = b. f = b / cb sub-blocks per tile side.

enum GemmMode : int {
  G_UPDATE_ALL = 0,  // column j: A_ik -= A_ij A_kj^T, j < k <= i   [K4/K5]
  G_UPDATE_COL = 1,  // column j: only k == j + 1  (lookahead part)
  G_UPDATE_REST = 2, // column j: only k >= j + 2
  G_PANEL_UPD = 3,   // column j, step c: A_ij[:,c] -= A_ij[:,<c] L_jj[c,<c]^T
  G_PANEL_TRSM = 4,  // column j, step c: A_ij[:,c]  = A_ij[:,c] W_jc^T   [K3]
  G_DIAG_TRSM = 5,   // column j, step s: D[r,s] = D[r,s] W_js^T, r > s
  G_DIAG_UPD = 6,    // column j, step s: D[r,c] -= D[r,s] D[c,s]^T, s<c<=r
  G_TRSM_X = 7,      // SIMT path: X_i = A_ij W_j^T into the panel buffer
  G_BATCH = 8,       // tests: C_t -= P_t Q_t^T (lower_only option)
  // distributed (2D block-cyclic) variants, items from host-built lists
  G_DIST_UPDATE = 9,      // owned (i, k): A_ik -= PB_i PB_k^T
  G_DIST_PANEL_UPD = 10,  // owned panel rows i: A_ij[:,c] -= A_ij[:,<c] Ld[c,<c]^T
  G_DIST_PANEL_TRSM = 11, // owned panel rows i: A_ij[:,c] = A_ij[:,c] Wb_c^T
  // column pairs (j, j1 = j + 1), K = 2b: A_ik -= [A_ij A_ij1] [A_kj A_kj1]^T
  // for tile column k = step only (k1 == step + 1) or every k >= step
  G_UPDATE_PAIR = 12,
  // distributed column pairs: owned (i, k) from the list, A / B rows from
  // the broadcast panel j (tensor map A) for k < b, then panel j + 1 (map B)
  G_DIST_UPDATE_PAIR = 13,
};

struct GemmArgs {
  int mode;
  int64_t j;        // column
  int step;         // c or s
  int64_t N;        // block rows
  int b, cb, f;
  double* A;        // packed tiles (local)
  int64_t tile_lo;
  const double* X;  // SIMT path panel buffer (tile i at (i - j - 1) b^2), or null
  double* Xout;
  const double* W;  // inverse blocks, block J at J * cb^2 (ld cb)
  double* C;        // batch outputs
  const double* P;  // batch operands
  const double* Q;
  int lower_only;
  const CholFlag* flag;
  const int64_t* lpos;    // cyclic layout: global tile -> local slot
  const int32_t* list;    // dist modes: (i, k) pairs or panel rows i
  int64_t k1;             // G_UPDATE_PAIR: step + 1 (one tile column) or N
};

struct GemmItem {
  const double* a;  // A_op: row 0, k 0 (ld = lda)
  const double* bp; // B_op
  int lda, ldb;
  int64_t a_tile, b_tile;  // TMA coordinates: tile index, row, k offset
  int a_r0, a_k0, b_r0, b_k0;
  // K = 2b column pairs: k-slices from k = b on come from these tiles
  int64_t a_tile2 = -1, b_tile2 = -1;
  bool two_maps = false;  // first half of K from map A, second from map B (both operands)
  double* c;        // output sub-block (ld = b)
  int K;
  int op;           // 0 SUB, 1 SET
  bool lower;
  bool skip;
};

__device__ __forceinline__ GemmItem decode_item(const GemmArgs& g, int64_t item) {
  GemmItem it{};
  const int b = g.b, cb = g.cb, f = g.f;
  const int64_t bb = (int64_t)b * b;
  auto tile = [&](int64_t i, int64_t k) {
    return g.lpos ? g.lpos[tri(i, k)] : tri(i, k) - g.tile_lo;
  };
  auto sub = [&](int64_t t, int r, int c) { return g.A + t * bb + (int64_t)r * cb * b + (int64_t)c * cb; };
  it.lda = it.ldb = b;
  it.op = 0;
  switch (g.mode) {
    case G_UPDATE_ALL:
    case G_UPDATE_COL:
    case G_UPDATE_REST: {
      const int64_t u = item / (f * f);
      const int sb = (int)(item % (f * f));
      const int mb = sb / f, nb = sb % f;
      int64_t i, k;
      if (g.mode == G_UPDATE_COL) {
        i = g.j + 1 + u;
        k = g.j + 1;
      } else {
        const int64_t base = g.mode == G_UPDATE_REST ? g.j + 2 : g.j + 1;
        const int64_t ii = tile_row(u);
        i = base + ii;
        k = base + (u - tri(ii, 0));
      }
      it.lower = (i == k) && mb == nb;
      it.skip = (i == k) && nb > mb;
      it.K = b;
      if (g.X) {  // SIMT path: panel in the buffer
        it.a = g.X + (i - g.j - 1) * bb + (int64_t)mb * cb * b;
        it.bp = g.X + (k - g.j - 1) * bb + (int64_t)nb * cb * b;
        it.a_tile = i - g.j - 1;
        it.b_tile = k - g.j - 1;
      } else {
        it.a = g.A + tile(i, g.j) * bb + (int64_t)mb * cb * b;
        it.bp = g.A + tile(k, g.j) * bb + (int64_t)nb * cb * b;
        it.a_tile = tile(i, g.j);
        it.b_tile = tile(k, g.j);
      }
      it.a_r0 = mb * cb;
      it.b_r0 = nb * cb;
      it.c = sub(tile(i, k), mb, nb);
      return it;
    }
    case G_UPDATE_PAIR: {
      const int64_t u = item / (f * f);
      const int sb = (int)(item % (f * f));
      const int mb = sb / f, nb = sb % f;
      int64_t i, k;
      if (g.k1 == g.step + 1) {
        k = g.step;
        i = k + u;
      } else {
        const int64_t ii = tile_row(u);
        i = g.step + ii;
        k = g.step + (u - tri(ii, 0));
      }
      it.lower = (i == k) && mb == nb;
      it.skip = (i == k) && nb > mb;
      it.K = 2 * b;
      it.a_tile = tile(i, g.j);
      it.b_tile = tile(k, g.j);
      it.a_tile2 = tile(i, g.j + 1);
      it.b_tile2 = tile(k, g.j + 1);
      it.a_r0 = mb * cb;
      it.b_r0 = nb * cb;
      it.c = sub(tile(i, k), mb, nb);
      return it;
    }
    case G_DIST_UPDATE_PAIR: {
      const int64_t u = item / (f * f);
      const int sb = (int)(item % (f * f));
      const int mb = sb / f, nb = sb % f;
      const int64_t i = g.list[2 * u], k = g.list[2 * u + 1];
      it.lower = (i == k) && mb == nb;
      it.skip = (i == k) && nb > mb;
      it.K = 2 * b;
      it.a_tile = i - g.j - 1;  // panel buffer of column j
      it.b_tile = k - g.j - 1;
      it.a_tile2 = i - g.j - 2; // panel buffer of column j + 1
      it.b_tile2 = k - g.j - 2;
      it.two_maps = true;
      it.a_r0 = mb * cb;
      it.b_r0 = nb * cb;
      it.c = sub(tile(i, k), mb, nb);
      return it;
    }
    case G_PANEL_UPD:
    case G_PANEL_TRSM: {
      const int64_t i = g.j + 1 + item / f;
      const int mb = (int)(item % f);
      const int c = g.step;
      it.a_tile = tile(i, g.j);
      it.a_r0 = mb * cb;
      it.c = sub(it.a_tile, mb, c);
      if (g.mode == G_PANEL_UPD) {
        it.a_k0 = 0;
        it.K = c * cb;
        it.b_tile = tile(g.j, g.j);
        it.b_r0 = c * cb;
        it.bp = g.A + it.b_tile * bb + (int64_t)c * cb * b;
      } else {
        it.a_k0 = c * cb;
        it.K = cb;
        it.b_tile = g.j * f + c;
        it.bp = g.W + it.b_tile * cb * cb;
        it.ldb = cb;
        it.op = 1;
      }
      it.a = g.A + it.a_tile * bb + (int64_t)it.a_r0 * b + it.a_k0;
      return it;
    }
    case G_DIAG_TRSM: {
      const int s = g.step, r = s + 1 + (int)item;
      it.a_tile = tile(g.j, g.j);
      it.a_r0 = r * cb;
      it.a_k0 = s * cb;
      it.a = g.A + it.a_tile * bb + (int64_t)it.a_r0 * b + it.a_k0;
      it.K = cb;
      it.b_tile = g.j * f + s;
      it.bp = g.W + it.b_tile * cb * cb;
      it.ldb = cb;
      it.c = sub(it.a_tile, r, s);
      it.op = 1;
      return it;
    }
    case G_DIAG_UPD: {
      const int s = g.step;
      const int ii = (int)tile_row(item), cc = (int)(item - tri(ii, 0));
      const int r = s + 1 + ii, c = s + 1 + cc;
      it.a_tile = it.b_tile = tile(g.j, g.j);
      it.a_r0 = r * cb;
      it.b_r0 = c * cb;
      it.a_k0 = it.b_k0 = s * cb;
      it.a = g.A + it.a_tile * bb + (int64_t)it.a_r0 * b + it.a_k0;
      it.bp = g.A + it.b_tile * bb + (int64_t)it.b_r0 * b + it.b_k0;
      it.K = cb;
      it.c = sub(it.a_tile, r, c);
      it.lower = (r == c);
      return it;
    }
    case G_TRSM_X: {  // SIMT path only (f == 1)
      const int64_t i = g.j + 1 + item;
      it.a = g.A + tile(i, g.j) * bb;
      it.bp = g.W + g.j * bb;
      it.K = b;
      it.c = g.Xout + (i - g.j - 1) * bb;
      it.op = 1;
      return it;
    }
    case G_DIST_UPDATE: {
      const int64_t u = item / (f * f);
      const int sb = (int)(item % (f * f));
      const int mb = sb / f, nb = sb % f;
      const int64_t i = g.list[2 * u], k = g.list[2 * u + 1];
      it.lower = (i == k) && mb == nb;
      it.skip = (i == k) && nb > mb;
      it.K = b;
      it.a_tile = i - g.j - 1;  // panel buffer tiles
      it.b_tile = k - g.j - 1;
      it.a = g.X + it.a_tile * bb + (int64_t)mb * cb * b;
      it.bp = g.X + it.b_tile * bb + (int64_t)nb * cb * b;
      it.a_r0 = mb * cb;
      it.b_r0 = nb * cb;
      it.c = sub(tile(i, k), mb, nb);
      return it;
    }
    case G_DIST_PANEL_UPD:
    case G_DIST_PANEL_TRSM: {
      const int64_t i = g.list[item / f];
      const int mb = (int)(item % f);
      const int c = g.step;
      it.a_tile = tile(i, g.j);
      it.a_r0 = mb * cb;
      it.c = sub(it.a_tile, mb, c);
      if (g.mode == G_DIST_PANEL_UPD) {
        it.a_k0 = 0;
        it.K = c * cb;
        it.b_tile = 0;  // the broadcast L_jj
        it.b_r0 = c * cb;
        it.bp = g.X + (int64_t)c * cb * b;
      } else {
        it.a_k0 = c * cb;
        it.K = cb;
        it.b_tile = c;  // the broadcast inverse blocks of L_jj
        it.bp = g.W + (int64_t)c * cb * cb;
        it.ldb = cb;
        it.op = 1;
      }
      it.a = g.A + it.a_tile * bb + (int64_t)it.a_r0 * b + it.a_k0;
      return it;
    }
    default: {  // G_BATCH
      const int64_t t = item / (f * f);
      const int sb = (int)(item % (f * f));
      const int mb = sb / f, nb = sb % f;
      it.a = g.P + t * bb + (int64_t)mb * cb * b;
      it.bp = g.Q + t * bb + (int64_t)nb * cb * b;
      it.a_tile = it.b_tile = t;
      it.a_r0 = mb * cb;
      it.b_r0 = nb * cb;
      it.K = b;
      it.c = g.C + t * bb + (int64_t)mb * cb * b + (int64_t)nb * cb;
      it.lower = g.lower_only && mb == nb;
      it.skip = g.lower_only && nb > mb;
      return it;
    }
  }
}

// ---------------------------------------------------------------------------
// DMMA sub-block GEMM (cb = 128), TMA-fed.

constexpr int GKS = 32, GSTAGES = 3;
// CTA tile BM x BN of an item's 128 x 128 output: 128 x 128 (the trailing
// updates), or split for launches of few items on the critical path (the
// diagonal-tile and panel steps; a 128^2 item with K = 128 takes ~23 us on
// one SM): 64 x 64 quadrants for C -= A B^T, 64 x 128 row halves for the
// in-place TRSM steps (C = A W^T with C = A: a CTA must read only the rows
// it writes)
template <int BM, int BN, int NST = GSTAGES>
struct GemmCfg {
  static constexpr int STAGES = NST;
  static constexpr int A_BYTES = BM * GKS * 8;
  static constexpr int B_BYTES = BN * GKS * 8;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int SMEM = NST * STAGE_BYTES + 1024 + 64;
  static constexpr int WM = BM / 32;      // warps along m (32 rows each)
  static constexpr int WN = 8 / WM;       // warps along n
  static constexpr int Y = BN / (WN * 8); // 8-column fragments per warp
};

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

template <int BM, int BN, int NST = GSTAGES>
__global__ void __launch_bounds__(288, 1)
    gemm_dmma_kernel(const __grid_constant__ CUtensorMap mapA,
                     const __grid_constant__ CUtensorMap mapB, GemmArgs g) {
  using Cfg = GemmCfg<BM, BN, NST>;
  constexpr int GSTAGES = NST;  // (shadows the default)
  constexpr int A_BYTES = Cfg::A_BYTES, B_BYTES = Cfg::B_BYTES;
  constexpr int G_STAGE_BYTES = Cfg::STAGE_BYTES;
  constexpr int GBM = BM, Y = Cfg::Y;
  if (g.flag && g.flag->status) return;
  // split tiles: part (qm, qn) of the item's 128 x 128 output
  constexpr int QM = 128 / BM, QN = 128 / BN;
  GemmItem it = decode_item(g, blockIdx.x / (QM * QN));
  int roff = 0, coff = 0;  // the tile's offset inside the item (lower test)
  if constexpr (QM * QN > 1) {
    const int part = (int)(blockIdx.x % (QM * QN)), qm = part / QN, qn = part % QN;
    roff = qm * BM;
    coff = qn * BN;
    if (it.lower && coff > roff + BM - 1) return;  // above a diagonal block's diagonal
    it.lower = it.lower && coff + BN - 1 > roff;  // straddles the diagonal
    it.a_r0 += roff;
    it.b_r0 += coff;
    it.c += (int64_t)roff * g.b + coff;
  }
  if (it.skip) return;
  const int nks = it.K / GKS;

  extern __shared__ __align__(1024) unsigned char gsm_raw[];
  // align by offsetting the shared pointer itself (a round trip through
  // uintptr_t would turn every operand load into a generic LD)
  unsigned char* gsm = gsm_raw + ((1024u - (smem_u32(gsm_raw) & 1023u)) & 1023u);
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
      for (int ks = 0; ks < nks; ++ks) {
        const int st = ks % GSTAGES;
        if (ks >= GSTAGES) mbar_wait(&empty[st], ((ks / GSTAGES) - 1) & 1);
        unsigned char* sa = gsm + st * G_STAGE_BYTES;
        unsigned char* sb = sa + A_BYTES;
        mbar_arrive_expect_tx(&full[st], G_STAGE_BYTES);
        int ka = it.a_k0 + ks * GKS, kb = it.b_k0 + ks * GKS;
        int at = (int)it.a_tile, bt = (int)it.b_tile;
        const CUtensorMap* ma = &mapA;
        const CUtensorMap* mbp = &mapB;
        if (it.a_tile2 >= 0 && ks * GKS >= g.b) {  // second column of a pair
          ka -= g.b;
          kb -= g.b;
          at = (int)it.a_tile2;
          bt = (int)it.b_tile2;
          if (it.two_maps) ma = &mapB;
        } else if (it.two_maps) {
          mbp = &mapA;
        }
        tma_load_3d(sa, ma, ka, it.a_r0, at, &full[st]);
        tma_load_3d(sa + A_BYTES / 2, ma, ka + 16, it.a_r0, at, &full[st]);
        tma_load_3d(sb, mbp, kb, it.b_r0, bt, &full[st]);
        tma_load_3d(sb + B_BYTES / 2, mbp, kb + 16, it.b_r0, bt, &full[st]);
      }
    }
    return;
  }

  // WM x WN warps of 32 x (8 Y): 4 x 2 of 32 x 64 (128 x 128), 2 x 4 of
  // 32 x 16 (64 x 64), 2 x 4 of 32 x 32 (64 x 128)
  const int wm = warp % Cfg::WM, wn = warp / Cfg::WM;
  double acc[4][Y][2];
#pragma unroll
  for (int x = 0; x < 4; ++x)
#pragma unroll
    for (int y = 0; y < Y; ++y) acc[x][y][0] = acc[x][y][1] = 0.0;
  const int fr = lane >> 2, fk = lane & 3;
  // Operand addresses, hoisted: element (row, k) of a [128 x 16] 128B-swizzled
  // box is at row*128 + ((k/2) ^ (row%8))*16 + (k%2)*8 (see swz). This
  // thread reads rows wm*32 + x*8 + fr (A) / wn*64 + y*8 + fr (B), so
  // row % 8 == fr, and k = 4 kk + fk. Only the XOR term depends on kk % 4;
  // x, y and kk / 4 become immediate offsets. (The half-warps' LDS.64 carry
  // a 2-way bank conflict in this order; a conflict-free row permutation
  // measured no faster -- the LSU pipe is < 10 % busy.)
  const uint32_t offA = (uint32_t)(wm * 32 + fr) * 128u + (uint32_t)(fk & 1) * 8u;
  const uint32_t offB = (uint32_t)(wn * 8 * Y + fr) * 128u + (uint32_t)(fk & 1) * 8u;
  uint32_t xo[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) xo[q] = (uint32_t)(((q * 2 + (fk >> 1)) ^ fr) << 4);

  for (int ks = 0; ks < nks; ++ks) {
    const int st = ks % GSTAGES;
    mbar_wait(&full[st], (ks / GSTAGES) & 1);
    const unsigned char* sa = gsm + st * G_STAGE_BYTES;
    const unsigned char* sb = sa + A_BYTES;
#pragma unroll
    for (int kk = 0; kk < GKS / 4; ++kk) {
      const uint32_t hA = (uint32_t)((kk >> 2) * (A_BYTES / 2)) + xo[kk & 3];
      const uint32_t hB = (uint32_t)((kk >> 2) * (B_BYTES / 2)) + xo[kk & 3];
      const double* pa = reinterpret_cast<const double*>(sa + offA + hA);
      const double* pb = reinterpret_cast<const double*>(sb + offB + hB);
      double af[4], bf[Y];
#pragma unroll
      for (int x = 0; x < 4; ++x) af[x] = pa[x * 128];  // + x * 1024 bytes
#pragma unroll
      for (int y = 0; y < Y; ++y) bf[y] = pb[y * 128];
#pragma unroll
      for (int x = 0; x < 4; ++x)
#pragma unroll
        for (int y = 0; y < Y; ++y) dmma_8x8x4(acc[x][y], af[x], bf[y]);
    }
    // the stage's operand reads (generic proxy) must be complete before the
    // TMA (async proxy) refills it. ptxas places the arrive right after the
    // last LDS, ahead of the DMMAs that consume them, so without this fence
    // (MEMBAR.CTA + FENCE.VIEW.ASYNC.S) the refill can overwrite data a
    // pending LDS has not read yet: wrong 64 x 64 tiles, two CTAs per SM,
    // when other work (copies, NCCL) loads the memory system
    // (tools/gpu/pollute_check.py; tools/sass_release_check.py checks the
    // SASS of every kernel for the pattern)
    fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[st]);
  }

  // epilogue: sub-block rows (wm*32 + x*8 + fr), cols (wn*8Y + y*8 + 2*fk)
  const int b = g.b;
  // (64 x 64 tiles too: 341.4 -> 340.3 ms at n = 32768, same bits -- C + (-acc)
  // == C - acc. Before the stage-release fence above existed they used a
  // plain read-modify-write, which made the stale-stage race rarer.)
  if ((BM == 128 || BN == 64) && it.op == 0 && !it.lower) {
    // C -= acc through the TMA engine: stage -acc row-major in the (now free)
    // stage buffers, then one bulk reduce-add per 1-KB row. The L2 performs
    // the read-modify-write; no register-held HBM round trips. (Per-element
    // red.global.add.f64 instead measured 1.4 % slower over a factorization.)
    named_bar_sync(1, 256);  // every MMA warp is done with the stage buffers
    constexpr int RS = BN * 8 + 16;  // padded smem row stride (bytes)
    unsigned char* tile = gsm;
#pragma unroll
    for (int x = 0; x < 4; ++x) {
      const int row = wm * 32 + x * 8 + fr;
#pragma unroll
      for (int y = 0; y < Y; ++y) {
        const int col = wn * 8 * Y + y * 8 + 2 * fk;
        *reinterpret_cast<double2*>(tile + row * RS + col * 8) =
            make_double2(-acc[x][y][0], -acc[x][y][1]);
      }
    }
    fence_proxy_async_smem();
    named_bar_sync(1, 256);
    if (tid < GBM) {
      bulk_reduce_add_f64(it.c + (int64_t)tid * b, tile + tid * RS, BN * 8);
      bulk_commit_group();
      bulk_wait_group_read0();
    }
    return;
  }
#pragma unroll
  for (int x = 0; x < 4; ++x) {
    const int row = wm * 32 + x * 8 + fr;
#pragma unroll
    for (int y = 0; y < Y; ++y) {
      const int col = wn * 8 * Y + y * 8 + 2 * fk;
      double2* p = reinterpret_cast<double2*>(it.c + (int64_t)row * b + col);
      if (it.op == 1) {
        *p = make_double2(acc[x][y][0], acc[x][y][1]);
      } else if (!it.lower || coff + col + 1 <= roff + row) {
        double2 v = *p;
        v.x -= acc[x][y][0];
        v.y -= acc[x][y][1];
        *p = v;
      } else if (coff + col <= roff + row) {
        it.c[(int64_t)row * b + col] -= acc[x][y][0];
      }
    }
  }
}

// ---------------------------------------------------------------------------
// SIMT FP64 sub-block GEMM (any cb): 64 x 64 CTA tiles over each item's
// cb x cb output, 4 x 4 per thread, K chunks of 16 staged in shared memory.
// Used only where cb % 128 != 0 (small / odd tile sizes), never in place
// across CTAs (G_TRSM_X writes the panel buffer).

__global__ void __launch_bounds__(256) gemm_simt_kernel(GemmArgs g) {
  if (g.flag && g.flag->status) return;
  const int cb = g.cb;
  const int tpd = (cb + 63) / 64;
  const int per = tpd * tpd;
  const int64_t item = blockIdx.x / per;
  const int sub = (int)(blockIdx.x % per);
  const int sm = sub / tpd, sn = sub % tpd;
  const GemmItem it = decode_item(g, item);
  if (it.skip) return;
  if (it.lower && sn > sm) return;
  __shared__ double As[16][65], Bs[16][65];
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  double acc[4][4];
#pragma unroll
  for (int x = 0; x < 4; ++x)
#pragma unroll
    for (int y = 0; y < 4; ++y) acc[x][y] = 0.0;
  const int m0 = sm * 64, n0 = sn * 64;
  for (int k0 = 0; k0 < it.K; k0 += 16) {
    for (int idx = threadIdx.x; idx < 64 * 16; idx += 256) {
      const int r = idx / 16, k = idx % 16;
      const int gr = m0 + r, gn = n0 + r, gk = k0 + k;
      As[k][r] = (gr < cb && gk < it.K) ? it.a[(int64_t)gr * it.lda + gk] : 0.0;
      Bs[k][r] = (gn < cb && gk < it.K) ? it.bp[(int64_t)gn * it.ldb + gk] : 0.0;
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
  const int b = g.b;
#pragma unroll
  for (int x = 0; x < 4; ++x)
#pragma unroll
    for (int y = 0; y < 4; ++y) {
      const int row = m0 + ty * 4 + x, col = n0 + tx * 4 + y;
      if (row >= cb || col >= cb) continue;
      if (it.lower && col > row) continue;
      double* p = it.c + (int64_t)row * b + col;
      if (it.op == 1) *p = acc[x][y];
      else *p -= acc[x][y];
    }
}

// ---------------------------------------------------------------------------
// diag128: POTRF + in-place TRTRI of one 128 x 128 diagonal sub-block held
// entirely in shared memory (256 threads), blocked in 32-wide panels so the
// CTA synchronises only a few times per panel:
//   factor, per panel p: warp 0 factors the 32x32 diagonal block; one thread
//     per row solves the panel rows below (x L^T = a, 32 registers); 4x4
//     register tiles apply the rank-32 update to the trailing triangle.
//   invert, panels right to left (LAPACK trtri order): one lane per column
//     inverts the 32x32 diagonal block; T = W_trail L_panel (scratch);
//     W_panel = -T W_pp.
// mode 0: factor + invert (the factorization's diagonal step; L is written
// back in place); mode 1: invert only (triangular solves on an uploaded
// factor; zero / NaN diagonal -> singular_block). W = L^-1 (zeros above the
// diagonal) goes to W + J*128^2.

constexpr int DCB = 128, DLD = 129, DPB = 32;
// S [128][129] | T scratch [96][33] | the four 32 x 32 diagonal-block inverses
// [4][32][33] (mode 0: formed while the other warps update, see below)
constexpr size_t kDiagSmemBytes =
    (size_t)(DCB * DLD + (DCB - DPB) * (DPB + 1) + (DCB / DPB) * DPB * (DPB + 1)) * 8;

// W = L^-1 of a 32 x 32 lower-triangular block by one warp, by rows in
// registers: lane r holds row r of L (a[]) and of W (w[]). Step k: lane k's
// row is final once scaled by 1 / L_kk and reaches the other lanes through
// shared memory (ck, double-buffered by step parity); every lane r > k then
// subtracts L_rk W_k,c -- the column recurrence
// W_rc = (delta_rc - sum_{c<=k<r} L_rk W_kc) / L_rr in the same k-ascending
// order, as independent chains across c. L at Lb (leading dimension ldl);
// the lower triangle of W goes to Wb (leading dimension ldw; may alias Lb).
__device__ __forceinline__ void diag_block_inverse(const double* Lb, int ldl, double* Wb, int ldw,
                                                   int lane, double* ck) {
  constexpr int NB = 32;
  double a[NB], w[NB];
#pragma unroll
  for (int c = 0; c < NB; ++c) {
    a[c] = c <= lane ? Lb[lane * ldl + c] : 0.0;
    w[c] = c == lane ? 1.0 : 0.0;
  }
#pragma unroll
  for (int k = 0; k < NB; ++k) {
    double* rowk = ck + (k & 1) * NB;
    if (lane == k) {
      const double rk = 1.0 / a[k];
#pragma unroll
      for (int c = 0; c <= k; ++c) {
        w[c] *= rk;
        rowk[c] = w[c];
      }
    }
    __syncwarp();
    // lanes > k subtract L_rk W_k,c; the others multiply by -0 (exact)
    const double lrk = lane > k ? a[k] : 0.0;
#pragma unroll
    for (int c = 0; c <= k; ++c) w[c] = fma(-lrk, rowk[c], w[c]);
  }
  __syncwarp();
#pragma unroll
  for (int c = 0; c < NB; ++c)
    if (c <= lane) Wb[lane * ldw + c] = w[c];
}

__global__ void __launch_bounds__(256)
    diag128_kernel(double* A, int64_t tile_lo, const int64_t* lpos, int b, int f,
                   double* W, int64_t J0, int mode, CholFlag* flag) {
  if (flag->status) return;
  const int64_t J = J0 + blockIdx.x;
  const int64_t j = J / f;
  const int sblk = (int)(J % f);
  const int64_t slot = lpos ? lpos[tri(j, j)] : tri(j, j) - tile_lo;
  double* D = A + slot * (int64_t)b * b + (int64_t)sblk * DCB * b + sblk * DCB;
  extern __shared__ double S[];       // [128][129]
  double* Tm = S + DCB * DLD;         // [96][33] scratch
  double* Wd = Tm + (DCB - DPB) * (DPB + 1);  // [4][32][33] W_pp = L_pp^-1
  __shared__ double Rv[DPB];          // reciprocal diagonal of the panel
  __shared__ __align__(16) double Ck[2 * DPB];  // warp 0's broadcast column / row
  __shared__ int bad;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
#pragma unroll 8
  for (int idx = tid; idx < DCB * DCB; idx += blockDim.x) {
    const int r = idx >> 7, c = idx & 127;
    S[r * DLD + c] = c <= r ? D[(int64_t)r * b + c] : 0.0;
  }
  if (tid == 0) bad = DCB;
  __syncthreads();
#ifdef HS_DIAG_TIMING
  __shared__ long long ts_clk[40];
  __shared__ const char* ts_name[40];
  int ts_n = 0;
  const long long ts0 = clock64();
#define HS_PHASE(name)                         \
  if (tid == 0 && ts_n < 40) {                 \
    ts_clk[ts_n] = clock64();                  \
    ts_name[ts_n++] = name;                    \
  }
#else
#define HS_PHASE(name)
#endif
  HS_PHASE("load");

  if (mode == 0) {
    for (int p = 0; p < DCB / DPB; ++p) {
      const int o = p * DPB;
      if (warp == 0) {
        // right-looking 32x32 factor in registers: lane r owns row r of the
        // block (fully unrolled, so a[] stays in registers); the pivot comes
        // from lane k and column k of L from the owning lanes by shuffle
        double* Dp = S + o * DLD + o;
        double a[DPB];
#pragma unroll
        for (int c = 0; c < DPB; ++c) a[c] = c <= lane ? Dp[lane * DLD + c] : 0.0;
        int failed = -1;
#pragma unroll
        for (int k = 0; k < DPB; ++k) {
          const double akk = __shfl_sync(0xffffffffu, a[k], k);
          // warp-uniform (broadcast pivot); no `break`, which would put a[]
          // in local memory
          if (failed < 0 && !(akk > 0.0)) failed = k;
          if (failed < 0) {
            // akk = +Inf passes the pivot test as in potf_block
            // (block_kernels.cpp:9-21): L_kk = sqrt(Inf) = Inf and the column
            // below is finite / Inf = 0 (rsqrt(Inf) = 0); akk * rinv would be
            // NaN there, so the diagonal takes akk itself
            const double rinv = rsqrt(akk);
            const double lrk = lane > k ? a[k] * rinv : 0.0;
            if (lane == k) a[k] = isinf(akk) ? akk : akk * rinv;
            if (lane > k) a[k] = lrk;
            // column k of L to every lane through a shared-memory broadcast
            // (double-buffered by step parity; 16-B loads), then the rank-1
            // update of this lane's row. Entries right of the diagonal
            // (c > lane) take garbage that is never read or stored; lanes
            // <= k have lrk = 0 and keep their rows
            double* colk = Ck + (k & 1) * DPB;
            colk[lane] = lrk;
            __syncwarp();
#pragma unroll
            for (int c = k + 1; c < DPB; ++c) a[c] = fma(-lrk, colk[c], a[c]);
          }
        }
        if (failed >= 0) {
          // the rows as far as the factorization got (the failing column's
          // pivot is reported; the tile is not used further)
          if (lane == 0) bad = o + failed;
        } else {
#pragma unroll
          for (int c = 0; c < DPB; ++c)
            if (c <= lane) Dp[lane * DLD + c] = a[c];
          __syncwarp();
          Rv[lane] = 1.0 / Dp[lane * DLD + lane];  // reciprocal diagonal
        }
      }
      __syncthreads();
      HS_PHASE("warpfactor");
      if (bad < DCB) {
        if (tid == 0) raise_flag(flag, HS_ERR_NOT_SPD, j, (int64_t)sblk * DCB + bad);
        return;
      }
      const int q0 = o + DPB, m = DCB - q0;
      if (warp == 0) {
        // W_pp = L_pp^-1 now, beside the other warps' panel solve and
        // update (the inverse pass below only copies it)
        diag_block_inverse(S + o * DLD + o, DLD, Wd + p * DPB * (DPB + 1), DPB + 1, lane, Ck);
      } else {
      const int t0 = tid - 32, nt = (int)blockDim.x - 32;
      // panel rows below: x L_pp^T = a
      for (int r = t0; r < m; r += nt) {
        double* row = S + (q0 + r) * DLD + o;
        double x[DPB];
#pragma unroll
        for (int c = 0; c < DPB; ++c) x[c] = row[c];
#pragma unroll
        for (int c = 0; c < DPB; ++c) {
          double acc = x[c];
#pragma unroll
          for (int k = 0; k < c; ++k) acc = fma(-x[k], S[(o + c) * DLD + o + k], acc);
          x[c] = acc * Rv[c];
        }
#pragma unroll
        for (int c = 0; c < DPB; ++c) row[c] = x[c];
      }
      named_bar_sync(2, nt);
      HS_PHASE("paneltrsm");
      // trailing rank-32 update of the lower triangle, 4x4 register tiles
      const int mt = m / 4, ntile = mt * (mt + 1) / 2;
      for (int u = t0; u < ntile; u += nt) {
        const int ti = (int)tile_row(u), tj = u - (int)tri(ti, 0);
        const int r0 = q0 + ti * 4, c0 = q0 + tj * 4;
        double acc[4][4] = {};
#pragma unroll 8
        for (int k = 0; k < DPB; ++k) {
          double a4[4], b4[4];
#pragma unroll
          for (int x = 0; x < 4; ++x) {
            a4[x] = S[(r0 + x) * DLD + o + k];
            b4[x] = S[(c0 + x) * DLD + o + k];
          }
#pragma unroll
          for (int x = 0; x < 4; ++x)
#pragma unroll
            for (int y = 0; y < 4; ++y) acc[x][y] = fma(a4[x], b4[y], acc[x][y]);
        }
#pragma unroll
        for (int x = 0; x < 4; ++x)
#pragma unroll
          for (int y = 0; y < 4; ++y)
            if (c0 + y <= r0 + x) S[(r0 + x) * DLD + c0 + y] -= acc[x][y];
      }
      }  // warps 1..7
      __syncthreads();
      HS_PHASE("update");
    }
    for (int idx = tid; idx < DCB * DCB; idx += blockDim.x) {
      const int r = idx >> 7, c = idx & 127;
      if (c <= r) D[(int64_t)r * b + c] = S[r * DLD + c];
    }
    // every thread has read the factor out of S before the inverse pass
    // overwrites it (its first step copies W_33 from Wd into S; compute-
    // sanitizer racecheck flagged the missing barrier)
    __syncthreads();
  } else {
    for (int r = tid; r < DCB; r += blockDim.x) {
      const double d = S[r * DLD + r];
      if (d == 0.0 || isnan(d)) atomicMin(&bad, r);
    }
    __syncthreads();
    if (bad < DCB) {
      if (tid == 0) raise_flag(flag, HS_ERR_SINGULAR_BLOCK, j, (int64_t)sblk * DCB + bad);
      return;
    }
  }

  // blocked in-place inverse, panels right to left
  for (int p = DCB / DPB - 1; p >= 0; --p) {
    const int o = p * DPB, q0 = o + DPB, m = DCB - q0;
    // (1) T = W_trail L_panel  (W_trail already inverted in place, lower;
    //     the strict upper part of S is zero, so k runs over full tiles)
    //     4x4 register tiles: 16 independent FMA chains per thread
    for (int u = tid; u < (m / 4) * (DPB / 4); u += blockDim.x) {
      const int r0 = (u / (DPB / 4)) * 4, c0 = (u % (DPB / 4)) * 4;
      double acc[4][4] = {};
      const int kend = r0 + 4;
#pragma unroll 4
      for (int k = 0; k < kend; ++k) {
        double w4[4], l4[4];
#pragma unroll
        for (int x = 0; x < 4; ++x) w4[x] = S[(q0 + r0 + x) * DLD + q0 + k];
#pragma unroll
        for (int y = 0; y < 4; ++y) l4[y] = S[(q0 + k) * DLD + o + c0 + y];
#pragma unroll
        for (int x = 0; x < 4; ++x)
#pragma unroll
          for (int y = 0; y < 4; ++y) acc[x][y] = fma(w4[x], l4[y], acc[x][y]);
      }
#pragma unroll
      for (int x = 0; x < 4; ++x)
#pragma unroll
        for (int y = 0; y < 4; ++y) Tm[(r0 + x) * (DPB + 1) + c0 + y] = acc[x][y];
    }
    HS_PHASE("inv_T");
    // (2) lane c inverts column c of the 32x32 diagonal block (registers)
    if (mode == 0) {
      // formed during the factorization (Wd)
      for (int idx = tid; idx < DPB * DPB; idx += blockDim.x) {
        const int r = idx >> 5, c = idx & 31;
        if (c <= r) S[(o + r) * DLD + o + c] = Wd[p * DPB * (DPB + 1) + r * (DPB + 1) + c];
      }
    } else if (warp == 0) {
      diag_block_inverse(S + o * DLD + o, DLD, S + o * DLD + o, DLD, lane, Ck);
    }
    __syncthreads();
    HS_PHASE("inv_diag");
    // (3) W_panel = -T W_pp  (W_pp lower; its upper part in S is zero)
    for (int u = tid; u < (m / 4) * (DPB / 4); u += blockDim.x) {
      const int r0 = (u / (DPB / 4)) * 4, c0 = (u % (DPB / 4)) * 4;
      double acc[4][4] = {};
#pragma unroll 8
      for (int k = c0; k < DPB; ++k) {
        double t4[4], w4[4];
#pragma unroll
        for (int x = 0; x < 4; ++x) t4[x] = Tm[(r0 + x) * (DPB + 1) + k];
#pragma unroll
        for (int y = 0; y < 4; ++y) w4[y] = S[(o + k) * DLD + o + c0 + y];
#pragma unroll
        for (int x = 0; x < 4; ++x)
#pragma unroll
          for (int y = 0; y < 4; ++y) acc[x][y] = fma(t4[x], w4[y], acc[x][y]);
      }
#pragma unroll
      for (int x = 0; x < 4; ++x)
#pragma unroll
        for (int y = 0; y < 4; ++y) S[(q0 + r0 + x) * DLD + o + c0 + y] = -acc[x][y];
    }
    __syncthreads();
    HS_PHASE("inv_panel");
  }
  double* Wj = W + J * DCB * DCB;
  for (int idx = tid; idx < DCB * DCB; idx += blockDim.x) {
    const int r = idx >> 7, c = idx & 127;
    Wj[idx] = c <= r ? S[r * DLD + c] : 0.0;
  }
  HS_PHASE("store");
#ifdef HS_DIAG_TIMING
  if (tid == 0 && blockIdx.x == 0 && J0 == 0) {
    long long prev = ts0;
    for (int k = 0; k < ts_n; ++k) {
      printf("diag128 %-12s %8lld\n", ts_name[k], ts_clk[k] - prev);
      prev = ts_clk[k];
    }
    printf("diag128 TOTAL %lld cycles\n", prev - ts0);
  }
#endif
}
#undef HS_PHASE

// ---------------------------------------------------------------------------
// small kernels

// A_ij <- X_i for i in (j, N)  (SIMT path)
__global__ void copy_panel_kernel(double* A, int64_t tile_lo, const double* X,
                                  int64_t j, int b, const CholFlag* flag) {
  if (flag->status) return;
  const int64_t i = j + 1 + blockIdx.y;
  const int64_t bb = (int64_t)b * b;
  const double* src = X + (i - j - 1) * bb;
  double* dst = A + (tri(i, j) - tile_lo) * bb;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < bb;
       k += (int64_t)gridDim.x * blockDim.x)
    dst[k] = src[k];
}

// NaN/Inf scan of the lower triangles (cholesky_solver.cpp:222-238): one
// warp per tile row, lanes over columns, no divisions in the inner loop.
__global__ void check_finite_kernel(const double* A, int64_t tile_lo,
                                    const int64_t* owned, int64_t ntiles, int b,
                                    CholFlag* flag) {
  const int64_t bb = (int64_t)b * b;
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  bool badv = false;
  int64_t bad_t = 0;
  for (int64_t w = warp; w < ntiles * b; w += nwarps) {
    const int64_t t = w / b;
    const int r = (int)(w - t * b);
    const int64_t gt = owned ? owned[t] : tile_lo + t;
    const int64_t i = tile_row(gt);
    const bool diag = (gt - tri(i, 0)) == i;
    const int cols = diag ? r + 1 : b;
    const double* row = A + t * bb + (int64_t)r * b;
    for (int c = lane; c < cols; c += 32)
      if (!isfinite(row[c])) {
        badv = true;
        bad_t = gt;
      }
  }
  if (badv) {
    const int64_t i = tile_row(bad_t);
    raise_flag(flag, HS_ERR_NUMERICAL, i, bad_t - tri(i, 0));
  }
}

// ---- triangular solves with the stored inverses ----------------------------
// Right-looking at tile granularity, 2 launches per tile row (PDL-chained):
//   forward  (L y = v):   y_i = solve(L_ii, v_i)   [trsv_diag_kernel, 8-CTA cluster]
//                         v_k -= L_ki y_i, k > i   [trsv_update_kernel]
//   backward (L^T x = v): x_i = solve(L_ii^T, v_i)
//                         v_k -= L_ik^T x_i, k < i
// The diagonal tile solve walks its f = b / cb sub-blocks with the stored
// cb x cb inverses W (cb = 128 on the DMMA path, b otherwise).

// v_i <- L_ii^-1 v_i (forward) or L_ii^-T v_i (backward) by a cluster of
// TRSV_CLUSTER CTAs (the diagonal solve is the substitutions' serial critical
// path: one CTA alone is load-latency bound at ~50 us for a 512 tile). Every
// CTA keeps full copies of vin / sol in its shared memory; per sub-block each
// CTA computes its share of the rows (forward) or columns (backward) and
// stores the new values into every CTA's copy through distributed shared
// memory, then a cluster barrier publishes them.
constexpr int TRSV_DIAG_THREADS = 512;
constexpr int TRSV_CLUSTER = 8;

__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\t"
               "barrier.cluster.wait.acquire.aligned;" ::: "memory");
}

__device__ __forceinline__ unsigned cluster_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

// store v at `p` (a shared-memory address of this CTA's layout) in all CTAs
__device__ __forceinline__ void st_cluster_all(double* p, double v) {
  const uint32_t a = smem_u32(p);
#pragma unroll
  for (int r = 0; r < TRSV_CLUSTER; ++r) {
    uint32_t ra;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(a), "r"(r));
    asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(ra), "d"(v) : "memory");
  }
}

// Staged variant (cb = 128 = TRSV_CLUSTER x 16 warps, f <= 4): each CTA's
// share of L_ii and of the inverses -- 16 rows (forward) or 16 columns
// (backward) per sub-block -- is copied into shared memory with cp.async
// before the PDL wait (the factor is constant), overlapping the previous
// update kernel; the sub-block steps then read shared memory only.
__host__ __device__ inline bool trsv_staged(int b, int cb, int f) {
  return cb == 128 && f <= 4 && b == cb * f;
}
// doubles staged per CTA: L_ii part 16 cb f(f-1)/2, inverses 16 cb f
__host__ __device__ inline int trsv_staged_doubles(int cb, int f) {
  return 16 * cb * (f * (f - 1) / 2 + f);
}

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src)
               : "memory");
}

// The sub-block steps of a diagonal-tile solve (vin holds the right-hand
// side in every CTA of the cluster; sol receives the solution in every CTA).
__device__ __forceinline__ void trsv_diag_steps(const double* D, const double* W, double* vin,
                                                double* sol, const double* Ds, const double* Ws,
                                                double (*red)[17], int b, int cb, int f,
                                                int64_t i, int upper, bool staged, int rank) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  // backward: 16 columns per group, nrl row lanes
  const int cg = tid & 15, rl = tid >> 4, nrl = blockDim.x >> 4;
  for (int step = 0; step < f; ++step) {
    const int sb = upper ? f - 1 - step : step;  // sub-block being solved
    const int o = sb * cb;
    // residual of sub-block sb: vin_sb - sum over solved sub-blocks
    //   forward:  L[sb][s'] sol_s' for s' < sb  (rows o.., cols < o)
    //   backward: L[s'][sb]^T sol_s' for s' > sb (rows > o+cb, cols o..)
    if (staged) {
      // forward: row warp of this CTA's 16; backward: column cg of its 16.
      // Sub-block sb's part of L_ii starts at 16 cb * (sum over s < sb of
      // s (forward) or f - 1 - s (backward) row-blocks)
      const int64_t dbase = upper ? 16LL * cb * (sb * (f - 1) - sb * (sb - 1) / 2)
                                  : 16LL * cb * (sb * (sb - 1) / 2);
      if (!upper && o > 0) {
        const double* row = Ds + dbase + warp * o;
        double a[4] = {0.0, 0.0, 0.0, 0.0};
        for (int c = lane; c < o; c += 128)
#pragma unroll
          for (int u = 0; u < 4; ++u) a[u] = fma(row[c + 32 * u], sol[c + 32 * u], a[u]);
        double acc = (a[0] + a[1]) + (a[2] + a[3]);
        for (int off = 16; off; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
        const int r = rank * 16 + warp;
        const double nv = vin[o + r] - acc;
        if (lane == 0) st_cluster_all(&vin[o + r], nv);
        cluster_sync_all();
      } else if (upper && o + cb < b) {
        const int nr = b - o - cb;
        double a0 = 0.0;
        for (int rr = rl; rr < nr; rr += nrl) a0 = fma(Ds[dbase + rr * 16 + cg], sol[o + cb + rr], a0);
        red[rl][cg] = a0;
        __syncthreads();
        if (rl == 0) {
          double t = 0.0;
          for (int p = 0; p < nrl; ++p) t += red[p][cg];
          const int c = o + rank * 16 + cg;
          st_cluster_all(&vin[c], vin[c] - t);
        }
        cluster_sync_all();
      }
    } else if (!upper) {
      if (o > 0) {
        for (int r = rank * nw + warp; r < cb; r += TRSV_CLUSTER * nw) {
          // 8 independent partial sums keep the row's loads in flight
          double a[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) a[u] = 0.0;
          const double* row = D + (int64_t)(o + r) * b;
          int c = lane;
          for (; c + 224 < o; c += 256)
#pragma unroll
            for (int u = 0; u < 8; ++u) a[u] = fma(row[c + 32 * u], sol[c + 32 * u], a[u]);
          for (; c < o; c += 32) a[0] = fma(row[c], sol[c], a[0]);
          double acc = ((a[0] + a[1]) + (a[2] + a[3])) + ((a[4] + a[5]) + (a[6] + a[7]));
          for (int off = 16; off; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
          const double nv = vin[o + r] - acc;
          if (lane == 0) st_cluster_all(&vin[o + r], nv);
        }
        cluster_sync_all();
      }
    } else {
      if (o + cb < b) {
        for (int c0 = 16 * rank; c0 < cb; c0 += 16 * TRSV_CLUSTER) {
          const int cc = c0 + cg;
          double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
          if (cc < cb) {
            const int c = o + cc;
            int r = o + cb + rl;
            for (; r + 3 * nrl < b; r += 4 * nrl) {
              a0 = fma(D[(int64_t)r * b + c], sol[r], a0);
              a1 = fma(D[(int64_t)(r + nrl) * b + c], sol[r + nrl], a1);
              a2 = fma(D[(int64_t)(r + 2 * nrl) * b + c], sol[r + 2 * nrl], a2);
              a3 = fma(D[(int64_t)(r + 3 * nrl) * b + c], sol[r + 3 * nrl], a3);
            }
            for (; r < b; r += nrl) a0 = fma(D[(int64_t)r * b + c], sol[r], a0);
          }
          red[rl][cg] = (a0 + a1) + (a2 + a3);
          __syncthreads();
          if (rl == 0 && cc < cb) {
            double t = 0.0;
            for (int p = 0; p < nrl; ++p) t += red[p][cg];
            st_cluster_all(&vin[o + cc], vin[o + cc] - t);
          }
          __syncthreads();
        }
        cluster_sync_all();
      }
    }
    // sol_sb = W_sb vin_sb (forward) or W_sb^T vin_sb (backward)
    const double* Wb = W + (i * f + sb) * (int64_t)cb * cb;
    if (staged) {
      if (!upper) {
        const int r = rank * 16 + warp;
        const double* wr = Ws + (sb * 16 + warp) * cb;
        double a[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int c = lane + 32 * u;
          if (c <= r) a[u] = wr[c] * vin[o + c];
        }
        double acc = (a[0] + a[1]) + (a[2] + a[3]);
        for (int off = 16; off; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
        if (lane == 0) st_cluster_all(&sol[o + r], acc);
      } else {
        const int c = rank * 16 + cg;
        double a0 = 0.0;
        for (int r = c + rl; r < cb; r += nrl) a0 = fma(Ws[(sb * cb + r) * 16 + cg], vin[o + r], a0);
        red[rl][cg] = a0;
        __syncthreads();
        if (rl == 0) {
          double t = 0.0;
          for (int p = 0; p < nrl; ++p) t += red[p][cg];
          st_cluster_all(&sol[o + c], t);
        }
        __syncthreads();
      }
    } else if (!upper) {
      for (int r = rank * nw + warp; r < cb; r += TRSV_CLUSTER * nw) {
        double a[4] = {0.0, 0.0, 0.0, 0.0};
        int c = lane;
        for (; c + 96 <= r; c += 128)
#pragma unroll
          for (int u = 0; u < 4; ++u)
            a[u] = fma(Wb[(int64_t)r * cb + c + 32 * u], vin[o + c + 32 * u], a[u]);
        for (; c <= r; c += 32) a[0] = fma(Wb[(int64_t)r * cb + c], vin[o + c], a[0]);
        double acc = (a[0] + a[1]) + (a[2] + a[3]);
        for (int off = 16; off; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
        if (lane == 0) st_cluster_all(&sol[o + r], acc);
      }
    } else {
      for (int c0 = 16 * rank; c0 < cb; c0 += 16 * TRSV_CLUSTER) {
        const int c = c0 + cg;
        double a0 = 0.0, a1 = 0.0;
        if (c < cb) {
          int r = c + rl;
          for (; r + nrl < cb; r += 2 * nrl) {
            a0 = fma(Wb[(int64_t)r * cb + c], vin[o + r], a0);
            a1 = fma(Wb[(int64_t)(r + nrl) * cb + c], vin[o + r + nrl], a1);
          }
          for (; r < cb; r += nrl) a0 = fma(Wb[(int64_t)r * cb + c], vin[o + r], a0);
        }
        red[rl][cg] = a0 + a1;
        __syncthreads();
        if (rl == 0 && c < cb) {
          double t = 0.0;
          for (int p = 0; p < nrl; ++p) t += red[p][cg];
          st_cluster_all(&sol[o + c], t);
        }
        __syncthreads();
      }
    }
    cluster_sync_all();
  }
}

__global__ void __launch_bounds__(TRSV_DIAG_THREADS)
    trsv_diag_kernel(const double* A, int64_t tile_lo, const int64_t* lpos, const double* W,
                     double* v, const double* G, int world, int b, int cb, int f, int64_t i,
                     int upper) {
  extern __shared__ double sh[];  // vin[b] | sol[b] | staged L_ii | staged W
  double* vin = sh;
  double* sol = sh + b;
  __shared__ double red[TRSV_DIAG_THREADS / 16][17];
  const double* D = A + (lpos ? lpos[tri(i, i)] : tri(i, i) - tile_lo) * (int64_t)b * b;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  const int rank = (int)cluster_rank();
  const bool staged = trsv_staged(b, cb, f) && nw * TRSV_CLUSTER == cb;
  // first half of the cluster barrier that guarantees every CTA of the
  // cluster is running before any DSMEM store (the wait is below)
  asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
  double* Ds = sh + 2 * b;               // [sb] blocks, see below
  double* Ws = Ds + 16 * cb * (f * (f - 1) / 2);  // [sb][cb][16] or [sb][16][cb]
  if (staged) {
    const double* Wi = W + i * f * (int64_t)cb * cb;
    int64_t base = 0;
    for (int sb = 0; sb < f; ++sb) {
      const int o = sb * cb;
      if (!upper) {
        // rows rank*16 + rr of sub-block sb, columns [0, o): Ds[base + rr*o + c]
        const int h = o / 2;  // 16-B chunks per row
        for (int q = tid; q < 16 * h; q += blockDim.x) {
          const int rr = q / h, cc = 2 * (q % h);
          cp_async16(Ds + base + rr * o + cc, D + (int64_t)(o + rank * 16 + rr) * b + cc);
        }
        base += 16 * o;
        for (int q = tid; q < 16 * cb / 2; q += blockDim.x) {
          const int rr = q / (cb / 2), cc = 2 * (q % (cb / 2));
          cp_async16(Ws + (sb * 16 + rr) * cb + cc,
                     Wi + ((int64_t)sb * cb + rank * 16 + rr) * cb + cc);
        }
      } else {
        // rows [o + cb, b), columns o + rank*16 + [0, 16): Ds[base + rr*16 + c]
        const int nr = b - o - cb;
        for (int q = tid; q < nr * 8; q += blockDim.x) {
          const int rr = q >> 3, cc = 2 * (q & 7);
          cp_async16(Ds + base + rr * 16 + cc, D + (int64_t)(o + cb + rr) * b + o + rank * 16 + cc);
        }
        base += 16 * nr;
        for (int q = tid; q < cb * 8; q += blockDim.x) {
          const int r = q >> 3, cc = 2 * (q & 7);
          cp_async16(Ws + (sb * cb + r) * 16 + cc,
                     Wi + ((int64_t)sb * cb + r) * cb + rank * 16 + cc);
        }
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  pdl_wait();
  pdl_trigger();
  // multi-rank: v_i plus every rank's (negated) partial update, rank order
  for (int k = tid; k < b; k += blockDim.x) {
    double t = v[i * b + k];
    if (G)
      for (int r = 0; r < world; ++r) t += G[(int64_t)r * b + k];
    vin[k] = t;
  }
  if (staged) asm volatile("cp.async.wait_all;" ::: "memory");
  __syncthreads();
  // every CTA arrived at kernel entry, so this returns at once. Remote
  // stores before the first full barrier below only target sol (which the
  // initialisation above does not write); remote vin stores happen after
  // it, i.e. after every CTA's initialisation.
  asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
  trsv_diag_steps(D, W, vin, sol, Ds, Ws, red, b, cb, f, i, upper, staged, rank);
  if (rank == 0)
    for (int k = tid; k < b; k += blockDim.x) v[i * b + k] = sol[k];
}

// forward: out_k[rows] -= L_ki[rows, :] y_i for k = i+1 .. N-1 (blockIdx.y),
//          row chunks (blockIdx.x; trsv_chunks)
// backward: out_k[cols] -= L_ik[:, cols]^T x_i for k = 0 .. i-1, column chunks
// (single rank: out = v; multi-rank: k from this rank's owned-tile `list`,
// out = its partial-update vector)
__global__ void __launch_bounds__(256)
    trsv_update_kernel(const double* A, int64_t tile_lo, const int64_t* lpos,
                       const int32_t* list, const double* v, double* out, int b,
                       int64_t i, int upper) {
  const bool cl = upper == 2;  // launched in clusters (launch_trsv_update)
  if (!list && blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) {
    // single rank: the next step's diagonal tile into L2 (the factor is
    // constant), so the diagonal solve's serial load chain hits L2
    const int64_t nx = upper ? i - 1 : i + 1;
    // (forward: launched only when a row below i exists; backward: i >= 1)
    if (nx >= 0) {
      // the bulk prefetch needs a 16-B aligned start and size (odd b: tiles
      // start 8-B aligned)
      const uintptr_t a0 = (uintptr_t)(A + (tri(nx, nx) - tile_lo) * (int64_t)b * b);
      const uintptr_t a16 = (a0 + 15) & ~(uintptr_t)15;
      const int64_t bytes = ((int64_t)b * b * 8 - (int64_t)(a16 - a0)) & ~(int64_t)15;
      if (bytes > 0) bulk_prefetch_l2(reinterpret_cast<const void*>(a16), (uint32_t)bytes);
    }
  }
  // DSMEM stores below only after every CTA of the cluster has started
  if (cl) asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
  pdl_wait();
  pdl_trigger();
  const int64_t k = list ? (int64_t)list[blockIdx.y]
                         : upper ? (int64_t)blockIdx.y : i + 1 + blockIdx.y;
  const int o0 = blockIdx.x * 32;
  extern __shared__ double yi[];  // [b]
  __shared__ double red[8][33];
  for (int c = threadIdx.x; c < b; c += blockDim.x) yi[c] = v[i * b + c];
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if ((b & 1) == 0 && upper != 1) {
    // even b: 16-byte loads (rows of a tile are 16-B aligned)
    const double2* yi2 = reinterpret_cast<const double2*>(yi);
    const int b2 = b / 2;
    if (!upper) {
      // 8 rows per CTA (blockIdx.x), one per warp: a row's loads all in flight
      const double* T = A + (lpos ? lpos[tri(k, i)] : tri(k, i) - tile_lo) * (int64_t)b * b;
      const int r = blockIdx.x * 8 + warp;
      if (r >= b) return;
      const double2* R0 = reinterpret_cast<const double2*>(T + (int64_t)r * b);
      double a0 = 0.0, a1 = 0.0, c0 = 0.0, c1 = 0.0;
      int c2 = lane;
#pragma unroll 4
      for (; c2 + 32 < b2; c2 += 64) {
        const double2 p = R0[c2], q = R0[c2 + 32], y = yi2[c2], z = yi2[c2 + 32];
        a0 = fma(p.x, y.x, a0);
        a1 = fma(p.y, y.y, a1);
        c0 = fma(q.x, z.x, c0);
        c1 = fma(q.y, z.y, c1);
      }
      if (c2 < b2) {
        const double2 p = R0[c2], y = yi2[c2];
        a0 = fma(p.x, y.x, a0);
        a1 = fma(p.y, y.y, a1);
      }
      double u = (a0 + a1) + (c0 + c1);
      for (int off = 16; off; off >>= 1) u += __shfl_xor_sync(0xffffffffu, u, off);
      if (lane == 0) out[k * b + r] -= u;
    } else {
      // a cluster of TRSV_CLUSTER CTAs per 64-column chunk (32 double2
      // lanes): CTA `rg` sums its row group, the leader adds the groups'
      // partials in rank order (deterministic) from its shared memory
      const int chunk = blockIdx.x / TRSV_CLUSTER, rg = blockIdx.x % TRSV_CLUSTER;
      const double* T = A + (lpos ? lpos[tri(i, k)] : tri(i, k) - tile_lo) * (int64_t)b * b;
      const int c2 = chunk * 32 + lane;
      const int R = (b + TRSV_CLUSTER - 1) / TRSV_CLUSTER;
      const int rlo = rg * R, rhi = min(b, rlo + R);
      double2 acc = make_double2(0.0, 0.0), acc1 = make_double2(0.0, 0.0);
      if (c2 < b2) {
        const double2* T2 = reinterpret_cast<const double2*>(T) + c2;
        int r = rlo + warp;
#pragma unroll 4
        for (; r + 8 < rhi; r += 16) {
          const double2 p = T2[(int64_t)r * b2], q = T2[(int64_t)(r + 8) * b2];
          acc.x = fma(p.x, yi[r], acc.x);
          acc.y = fma(p.y, yi[r], acc.y);
          acc1.x = fma(q.x, yi[r + 8], acc1.x);
          acc1.y = fma(q.y, yi[r + 8], acc1.y);
        }
        if (r < rhi) {
          const double2 p = T2[(int64_t)r * b2];
          acc.x = fma(p.x, yi[r], acc.x);
          acc.y = fma(p.y, yi[r], acc.y);
        }
      }
      __shared__ double2 red2[8][32];
      __shared__ double2 grp[TRSV_CLUSTER][32];  // leader: the groups' partials
      red2[warp][lane] = make_double2(acc.x + acc1.x, acc.y + acc1.y);
      __syncthreads();
      asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
      if (warp == 0) {
        double2 t = make_double2(0.0, 0.0);
        for (int w = 0; w < 8; ++w) {
          t.x += red2[w][lane].x;
          t.y += red2[w][lane].y;
        }
        uint32_t ra;
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;"
                     : "=r"(ra) : "r"(smem_u32(&grp[rg][lane])), "r"(0));
        asm volatile("st.shared::cluster.v2.f64 [%0], {%1, %2};" ::"r"(ra), "d"(t.x), "d"(t.y)
                     : "memory");
      }
      cluster_sync_all();
      if (rg == 0 && warp == 0 && c2 < b2) {
        double2 t = make_double2(0.0, 0.0);
        for (int g = 0; g < TRSV_CLUSTER; ++g) {
          t.x += grp[g][lane].x;
          t.y += grp[g][lane].y;
        }
        out[k * b + 2 * c2] -= t.x;
        out[k * b + 2 * c2 + 1] -= t.y;
      }
    }
    return;
  }
  if (!upper) {
    const double* T = A + (lpos ? lpos[tri(k, i)] : tri(k, i) - tile_lo) * (int64_t)b * b;
    for (int rr = warp; rr < 32; rr += 8) {
      const int r = o0 + rr;
      if (r >= b) break;
      double acc = 0.0;
      for (int c = lane; c < b; c += 32) acc = fma(T[(int64_t)r * b + c], yi[c], acc);
      for (int off = 16; off; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
      if (lane == 0) out[k * b + r] -= acc;
    }
  } else {
    const double* T = A + (lpos ? lpos[tri(i, k)] : tri(i, k) - tile_lo) * (int64_t)b * b;
    const int c = o0 + lane;
    double acc = 0.0;
    if (c < b)
      for (int r = warp; r < b; r += 8) acc = fma(T[(int64_t)r * b + c], yi[r], acc);
    red[warp][lane] = acc;
    __syncthreads();
    if (warp == 0 && c < b) {
      double t = 0.0;
      for (int w = 0; w < 8; ++w) t += red[w][lane];
      out[k * b + c] -= t;
    }
  }
}

// update variant (the kernel's `upper` argument): 0 forward; backward 1
// (one CTA per 32 columns over the whole tile height) or, at even b when the
// step has few tiles, 2 (one cluster of TRSV_CLUSTER CTAs per 64 columns,
// each CTA a row group: more SMs per tile where variant 1 would leave most
// of the GPU idle and latency-bound)
static int trsv_mode(int b, bool upper, int64_t nk) {
  if (!upper) return 0;
  return ((b & 1) == 0 && nk * ((b + 63) / 64) <= 148) ? 2 : 1;
}

// CTAs per tile along x: forward 8 rows per CTA at even b (16-byte loads)
static int trsv_chunks(int b, int mode) {
  if (mode == 2) return (b + 63) / 64 * TRSV_CLUSTER;
  if (mode == 0 && (b & 1) == 0) return (b + 7) / 8;
  return (b + 31) / 32;
}

template <typename... Args>
static cudaError_t launch_trsv_update(int mode, dim3 grid, size_t smem,
                                      cudaStream_t st, Args&&... args) {
  if (mode == 2)
    return launch_pdl_cluster(trsv_update_kernel, grid, dim3(256), TRSV_CLUSTER, smem, st,
                              std::forward<Args>(args)...);
  return launch_pdl(trsv_update_kernel, grid, dim3(256), smem, st, std::forward<Args>(args)...);
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

// 3-D map over `ntiles` contiguous side x side tiles: box 16 (k) x 128 x 1.
static CUtensorMap tile_map1(const double* base, int side, int64_t ntiles, int rows) {
  CUtensorMap m;
  cuuint64_t dims[3] = {(cuuint64_t)side, (cuuint64_t)side,
                        (cuuint64_t)std::max<int64_t>(ntiles, 1)};
  cuuint64_t strides[2] = {(cuuint64_t)side * 8, (cuuint64_t)side * side * 8};
  cuuint32_t box[3] = {16, (cuuint32_t)rows, 1};
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

// The two box heights of the DMMA GEMM's operand tiles (128- and 64-row CTAs)
struct TileMaps {
  CUtensorMap m128, m64;
};
static TileMaps tile_map(const double* base, int side, int64_t ntiles) {
  return TileMaps{tile_map1(base, side, ntiles, 128), tile_map1(base, side, ntiles, 64)};
}

CUtensorMap make_tensor_map(CUtensorMapDataType type, const void* base, int rank,
                            const cuuint64_t* dims, const cuuint64_t* strides,
                            const cuuint32_t* box, CUtensorMapSwizzle swizzle) {
  CUtensorMap m;
  cuuint32_t es[5] = {1, 1, 1, 1, 1};
  CUresult r = encode_fn()(&m, type, (cuuint32_t)rank, const_cast<void*>(base), dims,
                           strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  HS_REQUIRE(r == CUDA_SUCCESS, HS_ERR_CUDA, "cuTensorMapEncodeTiled failed");
  return m;
}

static bool dmma_ok(int b) { return b % 128 == 0; }
static int compute_block(int b) { return dmma_ok(b) ? 128 : b; }

static void launch_gemm(hs_ctx* c, cudaStream_t s, const GemmArgs& g,
                        int64_t items, const TileMaps* ma,
                        const TileMaps* mb) {
  if (items <= 0) return;
  if (g.cb == 128 && ma && mb) {
    // CTA tiles: 64 x 64 quadrants of the 128^2 items (two CTAs per SM, so one
    // CTA's start-up and epilogue overlap the other's DMMA work, and the
    // panel chain's small launches find SMs sooner than behind 128^2 CTAs),
    // 64 x 128 row halves for the in-place TRSM steps; HS_GEMM64=0: 128 x 128
    // throughout, HS_GEMM64=2: split tiles only for launches of at most one
    // wave (and in-place always within that rule)
    static const int q64 = [] {
      const char* e = getenv("HS_GEMM64");
      return e ? atoi(e) : 1;
    }();
    const int sms = std::max(1, c->num_sms);
    const bool in_place = g.mode == G_PANEL_TRSM || g.mode == G_DIAG_TRSM ||
                          g.mode == G_DIST_PANEL_TRSM;
    // (with the trailing update on the INT8 tensor cores only the panel
    // chain runs here, beside the Ozaki GEMM: split tiles for small launches
    // only, 184 vs 187 ms at n = 32768)
    const int pol = (q64 == 1 && c->chol_slices > 0) ? 2 : q64;
    const bool split = pol != 0 && (items <= sms || pol == 1);
    if (split && in_place) {
      using C = GemmCfg<64, 128>;
      static std::atomic<uint64_t> attr64{0};
      HS_CUDA(smem_attr_once(gemm_dmma_kernel<64, 128>, C::SMEM, attr64));
      gemm_dmma_kernel<64, 128><<<(unsigned)(items * 2), 288, C::SMEM, s>>>(ma->m64, mb->m128, g);
    } else if (split) {
      using C = GemmCfg<64, 64>;
      static std::atomic<uint64_t> attr64{0};
      HS_CUDA(smem_attr_once(gemm_dmma_kernel<64, 64>, C::SMEM, attr64));
      gemm_dmma_kernel<64, 64><<<(unsigned)(items * 4), 288, C::SMEM, s>>>(ma->m64, mb->m64, g);
    } else {
      using C = GemmCfg<128, 128>;
      static std::atomic<uint64_t> attr{0};
      HS_CUDA(smem_attr_once(gemm_dmma_kernel<128, 128>, C::SMEM, attr));
      gemm_dmma_kernel<128, 128><<<(unsigned)items, 288, C::SMEM, s>>>(ma->m128, mb->m128, g);
    }
  } else {
    const int tpd = (g.cb + 63) / 64;
    gemm_simt_kernel<<<(unsigned)(items * tpd * tpd), 256, 0, s>>>(g);
  }
  HS_CUDA(cudaGetLastError());
  launch_count(c);
}

static size_t potrf_smem(int b) { return (size_t)(PNB * PLD + b * PLD) * 8; }
static size_t trtri_smem(int b) { return (size_t)(PNB * PLD + PNB * b) * 8; }
static const size_t kDiagSmem = kDiagSmemBytes;

static void set_simt_tile_attrs(int b);

static void set_tile_kernel_attrs(int b) {
  if (dmma_ok(b)) {
    HS_CUDA(cudaFuncSetAttribute(diag128_kernel,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)kDiagSmem));
    return;
  }
  set_simt_tile_attrs(b);
}

static void set_simt_tile_attrs(int b) {
  HS_REQUIRE(potrf_smem(b) <= 227 * 1024 && trtri_smem(b) <= 227 * 1024,
             HS_ERR_CONFIG,
             "block size not a multiple of 128 must be <= 640 for the tile kernels");
  HS_CUDA(cudaFuncSetAttribute(potrf_tile_kernel,
                               cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)potrf_smem(b)));
  HS_CUDA(cudaFuncSetAttribute(trtri_tile_kernel,
                               cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)trtri_smem(b)));
}

struct ColStreams {
  cudaStream_t p = nullptr, u = nullptr, u2 = nullptr;
  std::vector<cudaEvent_t> ev;
  ~ColStreams() {
    for (auto e : ev) cudaEventDestroy(e);
    if (p) cudaStreamDestroy(p);
    if (u) cudaStreamDestroy(u);
    if (u2) cudaStreamDestroy(u2);
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

// All ranks agree on a distributed factorization's outcome: one all-reduce
// (max) of a key that orders failures by column, earliest first (the
// column a sequential factorization would have stopped at; a rank that runs
// on past another's failure can only fail later), then status and pivot.
// d_buf: 3 device int64 (the ledger logs one 24-byte scalar all-reduce).
static CholFlag agree_on_flag(hs_ctx* c, CholFlag h, int64_t* d_buf) {
  int64_t st[3] = {-1, 0, 0};
  if (h.status)
    st[0] = ((int64_t)(0x7fffffff - h.col) << 32) | ((int64_t)h.status << 24) |
            (h.pivot & 0xffffff);
  HS_CUDA(cudaMemcpy(d_buf, st, sizeof(st), cudaMemcpyHostToDevice));
  comm_allreduce_max_i64(c, d_buf, 3, c->stream);
  HS_CUDA(cudaMemcpyAsync(st, d_buf, sizeof(st), cudaMemcpyDeviceToHost, c->stream));
  HS_CUDA(cudaStreamSynchronize(c->stream));
  CholFlag out{};
  if (st[0] >= 0) {
    out.col = 0x7fffffff - (st[0] >> 32);
    out.status = (int32_t)((st[0] >> 24) & 0xff);
    out.pivot = st[0] & 0xffffff;
  }
  return out;
}

static void throw_flag(const CholFlag& h) {
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
  if (h.status == HS_ERR_SINGULAR_BLOCK)
    throw Failure{HS_ERR_SINGULAR_BLOCK,
                  "triangular block has zero or NaN diagonal at index " +
                      std::to_string(h.pivot),
                  h.col, h.pivot};
  if (h.status != HS_OK) throw Failure{h.status, "factorization failed", h.col, h.pivot};
}

static void alloc_inverses(hs_matrix* m) {
  const int cb = compute_block((int)m->b);
  const int64_t nblk = (int64_t)m->N * ((int64_t)m->b / cb);
  if (!m->dinv) HS_CUDA(cudaMalloc(&m->dinv, nblk * cb * cb * sizeof(double)));
}

// In-place factorization of a single-rank matrix.
static void potrf_run_dist(hs_ctx* c, hs_matrix* m);

static void potrf_run(hs_ctx* c, hs_matrix* m) {
  if (c->distributed() && m->layout == 1) {  // multi-rank: 2D block-cyclic path
    potrf_run_dist(c, m);
    return;
  }
  HS_REQUIRE(c->world == 1, HS_ERR_CONFIG,
             "multi-GPU Cholesky needs a cyclic matrix (hs_matrix_create_cyclic)");
  const int b = (int)m->b;
  const int cb = compute_block(b), f = b / cb;
  const bool fast = dmma_ok(b);
  const int64_t N = (int64_t)m->N;
  const int64_t bb = (int64_t)b * b;
  set_tile_kernel_attrs(b);
  alloc_inverses(m);
  m->has_inv = false;
  CholFlag* flag = static_cast<CholFlag*>(ctx_scratch(c));  // slot 0
  double* X[2] = {nullptr, nullptr};
  const int64_t panel = std::max<int64_t>(N - 1, 1);
  if (!fast) {  // panel buffers of the SIMT path, persistent across calls
    const size_t sz[2] = {(size_t)(panel * bb) * sizeof(double),
                          (size_t)(panel * bb) * sizeof(double)};
    void* ws[2];
    ctx_workspace(c, 3, sz, 2, ws);
    X[0] = static_cast<double*>(ws[0]);
    X[1] = static_cast<double*>(ws[1]);
  }
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

  TileMaps mapA{}, mapW{};
  if (fast) {
    mapA = tile_map(m->d, b, (int64_t)m->local_tiles());
    mapW = tile_map(m->dinv, cb, N * f);
  }
  // trailing update on the INT8 tensor cores (emulated FP64) when selected
  const bool use_oz = fast && c->chol_slices > 0 && N > 1;
  OzPanel& oz = ctx_oz_panel(c);  // buffers persist across calls
  if (use_oz) oz.init(b, N, c->chol_slices, /*pairs=*/true);

  GemmArgs g{};
  g.N = N;
  g.b = b;
  g.cb = cb;
  g.f = f;
  g.A = m->d;
  g.tile_lo = m->tile_lo;
  g.W = m->dinv;
  g.flag = flag;

  // P-stream work for column j: diagonal tile, then the panel below it.
  // panel steps of column block s on their own high-priority stream (P2),
  // each as soon as diag128(s) is done, beside the diagonal chain's later
  // sub-blocks: step s needs W_js and L_jj[s, <s] (final once diag128(s)
  // ran), and the diagonal chain only touches blocks right of column s
  // (HS_CHOL_PANEL_OVERLAP=0: after the whole diagonal tile, on P)
  static const bool panel_overlap = [] {
    const char* e = getenv("HS_CHOL_PANEL_OVERLAP");
    return !(e && atoi(e) == 0);
  }();
  cudaStream_t p2 = nullptr;
  if (fast && panel_overlap && !c->distributed()) {
    HS_CUDA(cudaStreamCreateWithPriority(&p2, cudaStreamNonBlocking, hi_pri));
    HS_CUDA(cudaStreamWaitEvent(p2, start));
  }
  struct P2Guard {
    cudaStream_t s;
    ~P2Guard() {
      if (s) cudaStreamDestroy(s);
    }
  } p2_guard{p2};
  auto panel_work = [&](int64_t j) {
    const int64_t t = N - 1 - j;
    if (fast) {
      auto panel_step = [&](int cc, cudaStream_t st) {
        GemmArgs gp = g;
        gp.j = j;
        gp.step = cc;
        if (cc > 0) {
          gp.mode = G_PANEL_UPD;
          launch_gemm(c, st, gp, t * f, &mapA, &mapA);
        }
        gp.mode = G_PANEL_TRSM;
        launch_gemm(c, st, gp, t * f, &mapA, &mapW);
      };
      for (int s = 0; s < f; ++s) {
        diag128_kernel<<<1, 256, kDiagSmem, cs.p>>>(m->d, m->tile_lo, nullptr, b, f,
                                                    m->dinv, j * f + s, 0, flag);
        HS_CUDA(cudaGetLastError());
        launch_count(c);
        if (p2 && t > 0) {
          cudaEvent_t ds = cs.make();
          HS_CUDA(cudaEventRecord(ds, cs.p));
          HS_CUDA(cudaStreamWaitEvent(p2, ds));
          panel_step(s, p2);
        }
        if (s + 1 < f) {
          GemmArgs gd = g;
          gd.j = j;
          gd.step = s;
          gd.mode = G_DIAG_TRSM;
          launch_gemm(c, cs.p, gd, f - 1 - s, &mapA, &mapW);
          gd.mode = G_DIAG_UPD;
          const int64_t tt = f - 1 - s;
          launch_gemm(c, cs.p, gd, tt * (tt + 1) / 2, &mapA, &mapA);
        }
      }
      if (p2 && t > 0) {
        cudaEvent_t pe = cs.make();
        HS_CUDA(cudaEventRecord(pe, p2));
        HS_CUDA(cudaStreamWaitEvent(cs.p, pe));
      } else {
        for (int cc = 0; cc < f && t > 0; ++cc) panel_step(cc, cs.p);
      }
      // single-column slices feed the even column's lookahead update
      if (use_oz && t > 0 && j % 2 == 0)
        oz.slice(c, cs.p, m->d, m->tile_lo, N, j, &flag->status);
      return;
    }
    // SIMT path (b % 128 != 0): single-CTA tile kernels, panel via buffer
    double* djj = m->d + (tri(j, j) - m->tile_lo) * bb;
    potrf_tile_kernel<<<1, 256, potrf_smem(b), cs.p>>>(djj, 0, b, flag, j);
    HS_CUDA(cudaGetLastError());
    trtri_tile_kernel<<<1, 256, trtri_smem(b), cs.p>>>(m->d, m->tile_lo, m->dinv, b,
                                                       flag, j);
    HS_CUDA(cudaGetLastError());
    launch_count(c, 2);
    if (t > 0) {
      GemmArgs gt = g;
      gt.mode = G_TRSM_X;
      gt.j = j;
      gt.Xout = X[j & 1];
      launch_gemm(c, cs.p, gt, t, nullptr, nullptr);
      dim3 grid((unsigned)std::max<int64_t>(1, std::min<int64_t>(64, ceil_div(bb, 512))),
                (unsigned)t);
      copy_panel_kernel<<<grid, 256, 0, cs.p>>>(m->d, m->tile_lo, X[j & 1], j, b, flag);
      HS_CUDA(cudaGetLastError());
      launch_count(c);
    }
  };

  panel_work(0);
  if (use_oz) {
    // INT8 path, columns in pairs (j0, j1 = j0 + 1): the trailing update of a
    // pair runs as ONE K = 2b update, [L_i,j0 L_i,j1] [L_k,j0 L_k,j1]^T, which
    // halves the epilogue passes over C (the K = b kernel is epilogue-bound:
    // 61 -> 83 TF/s at K = 2b). Schedule (P: panel stream, U: lookahead
    // updates, U2: the bulk "rest" update):
    //   U : tile column j1 by column j0 alone (K = b)    -> P: panel j1,
    //       joint slices of (j0, j1)
    //   U : tile column j1+1 by the pair                 -> P: panel j1+1 (next j0)
    //   U : tile column j1+2 by the pair
    //   U2: tile columns >= j1+3 by the pair, overlapping the next pair's
    //       panels and lookahead; the next pair's U work waits for it
    HS_CUDA(cudaStreamCreateWithPriority(&cs.u2, cudaStreamNonBlocking, lo_pri));
    HS_CUDA(cudaStreamWaitEvent(cs.u2, start));
    static const bool oz_hi = [] {
      const char* e = getenv("HS_OZ_U_HIPRI");
      return !(e && atoi(e) == 0);
    }();
    if (oz_hi) {  // the lookahead updates ahead of the bulk (as the DMMA pairs)
      HS_CUDA(cudaStreamDestroy(cs.u));
      HS_CUDA(cudaStreamCreateWithPriority(&cs.u, cudaStreamNonBlocking, hi_pri));
      HS_CUDA(cudaStreamWaitEvent(cs.u, start));
    }
    cudaEvent_t rest_done = nullptr;
    for (int64_t j0 = 0; j0 < N; j0 += 2) {
      const int64_t j1 = j0 + 1;
      if (j1 >= N) break;
      cudaEvent_t p0 = cs.make();
      HS_CUDA(cudaEventRecord(p0, cs.p));
      HS_CUDA(cudaStreamWaitEvent(cs.u, p0));
      oz.update(c, cs.u, m->d, m->tile_lo, (int64_t)m->local_tiles(), N, j0, true,
                &flag->status);
      cudaEvent_t ucol = cs.make();
      HS_CUDA(cudaEventRecord(ucol, cs.u));
      HS_CUDA(cudaStreamWaitEvent(cs.p, ucol));
      panel_work(j1);
      if (j1 + 1 >= N) break;
      oz.slice_pair(c, cs.p, m->d, m->tile_lo, N, j0, &flag->status);
      cudaEvent_t p1 = cs.make();
      HS_CUDA(cudaEventRecord(p1, cs.p));
      HS_CUDA(cudaStreamWaitEvent(cs.u, p1));
      if (rest_done) HS_CUDA(cudaStreamWaitEvent(cs.u, rest_done));
      oz.update_pair(c, cs.u, m->d, m->tile_lo, N, j0, true, j1 + 1, &flag->status);
      cudaEvent_t ua = cs.make();
      HS_CUDA(cudaEventRecord(ua, cs.u));
      if (j1 + 2 < N) {
        oz.update_pair(c, cs.u, m->d, m->tile_lo, N, j0, true, j1 + 2, &flag->status);
        cudaEvent_t ub = cs.make();
        HS_CUDA(cudaEventRecord(ub, cs.u));
        if (j1 + 3 < N) {
          HS_CUDA(cudaStreamWaitEvent(cs.u2, ub));
          oz.update_pair(c, cs.u2, m->d, m->tile_lo, N, j0, false, j1 + 3, &flag->status);
          rest_done = cs.make();
          HS_CUDA(cudaEventRecord(rest_done, cs.u2));
        }
      }
      HS_CUDA(cudaStreamWaitEvent(cs.p, ua));
      panel_work(j1 + 1);
    }
  }
  // HS_CHOL_TIMING=1: per-column event times of the default schedule on
  // stderr (panel chain on P, column-(j+1) update and rest on U)
  static const bool col_timing = getenv("HS_CHOL_TIMING") != nullptr;
  std::vector<cudaEvent_t> tev;
  auto tmark = [&](cudaStream_t st) {
    if (!col_timing) return;
    cudaEvent_t e;
    HS_CUDA(cudaEventCreate(&e));
    HS_CUDA(cudaEventRecord(e, st));
    tev.push_back(e);
  };
  // DMMA in column pairs (the INT8 path's schedule above): the bulk of the
  // trailing update runs with K = 2b per CTA, halving the per-CTA start-up and
  // epilogue share of each 128^2 item (HS_CHOL_PAIRS=0: one column at a time)
  static const bool pairs_env = [] {
    const char* e = getenv("HS_CHOL_PAIRS");
    return !(e && atoi(e) == 0);
  }();
  const bool pairs = pairs_env && fast && !use_oz && N >= 4;
  if (pairs) {
    HS_CUDA(cudaStreamCreateWithPriority(&cs.u2, cudaStreamNonBlocking, lo_pri));
    HS_CUDA(cudaStreamWaitEvent(cs.u2, start));
    // the lookahead updates feed the panel chain: the panel's priority, so
    // they take SMs ahead of the bulk update on U2
    HS_CUDA(cudaStreamDestroy(cs.u));
    HS_CUDA(cudaStreamCreateWithPriority(&cs.u, cudaStreamNonBlocking, hi_pri));
    HS_CUDA(cudaStreamWaitEvent(cs.u, start));
    cudaEvent_t rest_done = nullptr;
    int64_t j0 = 0;
    for (; j0 + 1 < N; j0 += 2) {
      const int64_t j1 = j0 + 1;
      // tile column j1 by panel j0 alone, then panel j1
      // (tile column j1 is not in the previous pair's bulk, which covers
      // columns >= j1 + 2: that bulk keeps running beside this update and
      // both of this pair's panels)
      cudaEvent_t p0 = cs.make();
      HS_CUDA(cudaEventRecord(p0, cs.p));
      tmark(cs.p);
      HS_CUDA(cudaStreamWaitEvent(cs.u, p0));
      GemmArgs gu = g;
      gu.j = j0;
      gu.mode = G_UPDATE_COL;
      launch_gemm(c, cs.u, gu, (N - 1 - j0) * f * f, &mapA, &mapA);
      cudaEvent_t ucol = cs.make();
      HS_CUDA(cudaEventRecord(ucol, cs.u));
      tmark(cs.u);
      HS_CUDA(cudaStreamWaitEvent(cs.p, ucol));
      panel_work(j1);
      tmark(cs.p);
      if (j1 + 1 >= N) break;
      // columns > j1 by the pair (K = 2b): j1+1 first (the next panel needs
      // it), j1+2, then the bulk on U2 beside the next pair's panels
      cudaEvent_t p1 = cs.make();
      HS_CUDA(cudaEventRecord(p1, cs.p));
      HS_CUDA(cudaStreamWaitEvent(cs.u, p1));
      if (rest_done) HS_CUDA(cudaStreamWaitEvent(cs.u, rest_done));  // previous bulk
      GemmArgs gp = g;
      gp.j = j0;
      gp.mode = G_UPDATE_PAIR;
      gp.step = (int)(j1 + 1);
      gp.k1 = j1 + 2;
      launch_gemm(c, cs.u, gp, (N - 1 - j1) * f * f, &mapA, &mapA);
      cudaEvent_t ua = cs.make();
      HS_CUDA(cudaEventRecord(ua, cs.u));
      tmark(cs.u);
      rest_done = nullptr;
      if (j1 + 2 < N) {
        gp.step = (int)(j1 + 2);
        gp.k1 = j1 + 3;
        launch_gemm(c, cs.u, gp, (N - 2 - j1) * f * f, &mapA, &mapA);
        cudaEvent_t ub = cs.make();
        HS_CUDA(cudaEventRecord(ub, cs.u));
        if (j1 + 3 < N) {
          HS_CUDA(cudaStreamWaitEvent(cs.u2, ub));
          gp.step = (int)(j1 + 3);
          gp.k1 = N;
          const int64_t tr = N - 3 - j1;
          launch_gemm(c, cs.u2, gp, tr * (tr + 1) / 2 * f * f, &mapA, &mapA);
          rest_done = cs.make();
          HS_CUDA(cudaEventRecord(rest_done, cs.u2));
        }
      }
      tmark(cs.u2);
      HS_CUDA(cudaStreamWaitEvent(cs.p, ua));
      panel_work(j1 + 1);
      tmark(cs.p);
    }
    if (col_timing && !tev.empty()) {
      HS_CUDA(cudaDeviceSynchronize());
      auto ms = [&](size_t k) {
        float v = 0.f;
        cudaEventElapsedTime(&v, tev[0], tev[k]);
        return v;
      };
      fprintf(stderr, "chol pairs: j0 panel_j0_end ucol_end panel_j1_end ua_end bulk_end "
                      "panel_j1+1_end (ms)\n");
      for (size_t k = 0, j = 0; k + 6 <= tev.size(); k += 6, j += 2)
        fprintf(stderr, "pair %3zu %9.3f %9.3f %9.3f %9.3f %9.3f %9.3f\n", j, ms(k), ms(k + 1),
                ms(k + 2), ms(k + 3), ms(k + 4), ms(k + 5));
      for (cudaEvent_t e : tev) cudaEventDestroy(e);
      tev.clear();
    }
    // an odd trailing column: its panel j0 = N - 1 is the last one
  }
  // HS_CHOL_SCHED=1: the rest of column j's update runs on its own
  // low-priority stream from the moment the panel is done, next to the
  // high-priority column-(j+1) update (whose last wave it fills), instead of
  // after it on the same stream
  static const int sched = [] {
    const char* e = getenv("HS_CHOL_SCHED");
    return e ? atoi(e) : 0;
  }();
  if (sched == 1 && !use_oz && !pairs && N > 1) {
    HS_CUDA(cudaStreamCreateWithPriority(&cs.u2, cudaStreamNonBlocking, lo_pri));
    HS_CUDA(cudaStreamWaitEvent(cs.u2, start));
    HS_CUDA(cudaStreamDestroy(cs.u));  // re-created with the panel's priority
    HS_CUDA(cudaStreamCreateWithPriority(&cs.u, cudaStreamNonBlocking, hi_pri));
    HS_CUDA(cudaStreamWaitEvent(cs.u, start));
    for (int64_t j = 0; j + 1 < N; ++j) {
      const int64_t t = N - 1 - j;
      cudaEvent_t pdone = cs.make();
      HS_CUDA(cudaEventRecord(pdone, cs.p));
      GemmArgs gu = g;
      gu.j = j;
      gu.X = fast ? nullptr : X[j & 1];
      const TileMaps* mx = fast ? &mapA : nullptr;
      // column j+1 (urgent): after panel j and after REST(j-1), which
      // updated these tiles with panel j-1
      HS_CUDA(cudaStreamWaitEvent(cs.u, pdone));
      gu.mode = G_UPDATE_COL;
      launch_gemm(c, cs.u, gu, t * f * f, mx, mx);
      cudaEvent_t ucol = cs.make();
      HS_CUDA(cudaEventRecord(ucol, cs.u));
      // columns > j+1: alongside, low priority (u2 is in order with REST(j-1))
      HS_CUDA(cudaStreamWaitEvent(cs.u2, pdone));
      gu.mode = G_UPDATE_REST;
      const int64_t tr = t - 1;
      if (tr > 0) launch_gemm(c, cs.u2, gu, tr * (tr + 1) / 2 * f * f, mx, mx);
      cudaEvent_t rdone = cs.make();
      HS_CUDA(cudaEventRecord(rdone, cs.u2));
      HS_CUDA(cudaStreamWaitEvent(cs.u, rdone));  // before UCOL(j+1)
      HS_CUDA(cudaStreamWaitEvent(cs.p, ucol));
      panel_work(j + 1);
    }
  }
  cudaStream_t su = cs.u;
  if (!pairs) tmark(cs.p);
  for (int64_t j = 0; j < N && !use_oz && !pairs && sched != 1; ++j) {
    const int64_t t = N - 1 - j;
    cudaEvent_t pdone = cs.make();
    HS_CUDA(cudaEventRecord(pdone, cs.p));
    if (t == 0) break;
    HS_CUDA(cudaStreamWaitEvent(su, pdone));
    GemmArgs gu = g;
    gu.j = j;
    gu.X = fast ? nullptr : X[j & 1];
    const TileMaps* mx = fast ? &mapA : nullptr;
    // lookahead: tile column j+1 first
    tmark(su);
    gu.mode = G_UPDATE_COL;
    launch_gemm(c, su, gu, t * f * f, mx, mx);
    cudaEvent_t ucol = cs.make();
    HS_CUDA(cudaEventRecord(ucol, su));
    tmark(su);
    HS_CUDA(cudaStreamWaitEvent(cs.p, ucol));
    // the rest of column j's update overlaps column j+1's panel work (the
    // panel touches only tile column j+1; the update reads column j)
    gu.mode = G_UPDATE_REST;
    const int64_t tr = t - 1;
    launch_gemm(c, su, gu, tr * (tr + 1) / 2 * f * f, mx, mx);
    tmark(su);
    tmark(cs.p);
    panel_work(j + 1);
    tmark(cs.p);
  }
  if (col_timing && !tev.empty()) {
    HS_CUDA(cudaDeviceSynchronize());
    auto ms = [&](size_t k) {
      float v = 0.f;
      cudaEventElapsedTime(&v, tev[0], tev[k]);
      return v;
    };
    fprintf(stderr, "chol timing: j ucol_start ucol_end rest_end panel_start panel_end (ms)\n");
    for (size_t k = 1, j = 0; k + 4 < tev.size() + 1 && k + 4 <= tev.size(); k += 5, ++j)
      fprintf(stderr, "chol %3zu %9.3f %9.3f %9.3f %9.3f %9.3f\n", j, ms(k), ms(k + 1),
              ms(k + 2), ms(k + 3), ms(k + 4));
    for (cudaEvent_t e : tev) cudaEventDestroy(e);
  }
  cudaEvent_t pend = cs.make(), uend = cs.make();
  HS_CUDA(cudaEventRecord(pend, cs.p));
  HS_CUDA(cudaEventRecord(uend, cs.u));
  HS_CUDA(cudaStreamWaitEvent(c->stream, pend));
  HS_CUDA(cudaStreamWaitEvent(c->stream, uend));
  if (cs.u2) {
    cudaEvent_t u2end = cs.make();
    HS_CUDA(cudaEventRecord(u2end, cs.u2));
    HS_CUDA(cudaStreamWaitEvent(c->stream, u2end));
  }
  check_finite_kernel<<<4 * 148, 256, 0, c->stream>>>(
      m->d, m->tile_lo, nullptr, (int64_t)m->local_tiles(), b, flag);
  HS_CUDA(cudaGetLastError());
  launch_count(c);
  CholFlag h{};
  HS_CUDA(cudaMemcpyAsync(&h, flag, sizeof(h), cudaMemcpyDeviceToHost, c->stream));
  HS_CUDA(cudaStreamSynchronize(c->stream));
  throw_flag(h);
  m->has_inv = true;
}


// ---------------------------------------------------------------------------
// Distributed factorization: 2D block-cyclic tiles over a P x Q grid
// (hs_matrix_create_cyclic), one process per GPU, NCCL over NVLink.
// Per column j:
//   owner(j,j): POTRF/TRTRI of the diagonal tile (diag128 + DMMA GEMMs)
//   broadcast L_jj and its 128^2 inverse blocks to every rank
//   owners of panel tiles (i, j): in-place blocked TRSM (DMMA)
//   broadcast every panel tile from its owner into the panel buffer PB
//   every rank: A_ik -= PB_i PB_k^T on its own trailing tiles
// with the same one-column lookahead as the single-GPU path (P stream:
// diagonal, TRSM and all NCCL calls, in the same order on every rank; U
// stream: updates, the column j+1 tiles first).


static void potrf_run_dist(hs_ctx* c, hs_matrix* m) {
  const int b = (int)m->b;
  HS_REQUIRE(dmma_ok(b), HS_ERR_CONFIG,
             "distributed Cholesky needs a block size that is a multiple of 128");
  HS_REQUIRE(m->layout == 1, HS_ERR_CONFIG,
             "distributed Cholesky needs a cyclic matrix (hs_matrix_create_cyclic)");
  const int cb = 128, f = b / cb;
  const int64_t N = (int64_t)m->N;
  const int64_t bb = (int64_t)b * b;
  const int P = m->P, Q = m->Q, me = c->rank;
  set_tile_kernel_attrs(b);
  alloc_inverses(m);
  m->has_inv = false;

  // host work lists: per column, the owned panel rows and owned trailing
  // pairs (COL part k == j+1 first, then REST), concatenated
  std::vector<int32_t> rows, pairs;
  std::vector<int64_t> row_off(N + 1, 0), col_off(N + 1, 0), rest_off(N + 1, 0);
  for (int64_t j = 0; j < N; ++j) {
    row_off[j] = (int64_t)rows.size();
    for (int64_t i = j + 1; i < N; ++i)
      if (cyclic_owner(i, j, P, Q) == me) rows.push_back((int32_t)i);
    col_off[j] = (int64_t)pairs.size() / 2;
    for (int64_t i = j + 1; i < N; ++i)
      if (cyclic_owner(i, j + 1, P, Q) == me) {
        pairs.push_back((int32_t)i);
        pairs.push_back((int32_t)(j + 1));
      }
    rest_off[j] = (int64_t)pairs.size() / 2;
    for (int64_t i = j + 2; i < N; ++i)
      for (int64_t k = j + 2; k <= i; ++k)
        if (cyclic_owner(i, k, P, Q) == me) {
          pairs.push_back((int32_t)i);
          pairs.push_back((int32_t)k);
        }
  }
  row_off[N] = (int64_t)rows.size();
  col_off[N] = rest_off[N] = (int64_t)pairs.size() / 2;
  // column pairs (DMMA; HS_CHOL_PAIRS=0: one column at a time): per pair
  // (j0, j1 = j0 + 1) the owned (i, k) of tile column j1 + 1, of j1 + 2, and
  // of the columns beyond, updated with K = 2b from both broadcast panels
  static const bool dist_pairs_env = [] {
    const char* e = getenv("HS_CHOL_PAIRS");
    return !(e && atoi(e) == 0);
  }();
  const bool dpairs = dist_pairs_env && c->chol_slices == 0 && N >= 4;
  std::vector<int64_t> pp_off;  // 3 lists per pair: [4 m, 4 m + 3]
  if (dpairs) {
    for (int64_t j0 = 0; j0 + 1 < N; j0 += 2) {
      const int64_t j1 = j0 + 1;
      pp_off.push_back((int64_t)pairs.size() / 2);
      for (int64_t i = j1 + 1; i < N; ++i)
        if (cyclic_owner(i, j1 + 1, P, Q) == me) {
          pairs.push_back((int32_t)i);
          pairs.push_back((int32_t)(j1 + 1));
        }
      pp_off.push_back((int64_t)pairs.size() / 2);
      for (int64_t i = j1 + 2; i < N; ++i)
        if (cyclic_owner(i, j1 + 2, P, Q) == me) {
          pairs.push_back((int32_t)i);
          pairs.push_back((int32_t)(j1 + 2));
        }
      pp_off.push_back((int64_t)pairs.size() / 2);
      for (int64_t i = j1 + 3; i < N; ++i)
        for (int64_t k = j1 + 3; k <= i; ++k)
          if (cyclic_owner(i, k, P, Q) == me) {
            pairs.push_back((int32_t)i);
            pairs.push_back((int32_t)k);
          }
      pp_off.push_back((int64_t)pairs.size() / 2);
    }
  }

  const int64_t panel = std::max<int64_t>(N - 1, 1);
  CholFlag* flag = static_cast<CholFlag*>(ctx_scratch(c));  // slot 0
  int64_t* d_status = reinterpret_cast<int64_t*>(flag + 1);
  // panel broadcast buffers and work lists from the context's persistent
  // workspace (a per-call cudaMalloc / cudaFree of the ~250 MB at n=32768
  // stalls the host for tens of ms)
  // panel buffers: 2 (by column parity), 4 with column pairs (a pair's bulk
  // update reads both of its panels while the next pair's arrive)
  const int npb = dpairs ? 4 : 2;
  const size_t sz[8] = {std::max<size_t>(rows.size(), 1) * sizeof(int32_t),
                        std::max<size_t>(pairs.size(), 2) * sizeof(int32_t),
                        (size_t)bb * sizeof(double),
                        (size_t)f * cb * cb * sizeof(double),
                        (size_t)(panel * bb) * sizeof(double),
                        (size_t)(panel * bb) * sizeof(double),
                        dpairs ? (size_t)(panel * bb) * sizeof(double) : 0,
                        dpairs ? (size_t)(panel * bb) * sizeof(double) : 0};
  void* ws[8];
  ctx_workspace(c, 1, sz, 8, ws);
  int32_t* d_rows = static_cast<int32_t*>(ws[0]);
  int32_t* d_pairs = static_cast<int32_t*>(ws[1]);
  double* Ld = static_cast<double*>(ws[2]);
  double* Wb = static_cast<double*>(ws[3]);
  double* PB[4] = {static_cast<double*>(ws[4]), static_cast<double*>(ws[5]),
                   static_cast<double*>(ws[6]), static_cast<double*>(ws[7])};
  auto pbi = [&](int64_t j) { return (int)(j % npb); };
  if (!rows.empty())
    HS_CUDA(cudaMemcpy(d_rows, rows.data(), rows.size() * sizeof(int32_t),
                       cudaMemcpyHostToDevice));
  if (!pairs.empty())
    HS_CUDA(cudaMemcpy(d_pairs, pairs.data(), pairs.size() * sizeof(int32_t),
                       cudaMemcpyHostToDevice));
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
  cudaStream_t cs_u = cs.u;

  const TileMaps mapA = tile_map(m->d, b, std::max<int64_t>((int64_t)m->local_tiles(), 1));
  const TileMaps mapW = tile_map(m->dinv, cb, N * f);
  // trailing update on the INT8 tensor cores when selected (slices of the
  // broadcast panel, double buffered like PB)
  const bool use_oz = c->chol_slices > 0 && N > 1;
  OzPanel& oz = ctx_oz_panel(c);  // buffers persist across calls
  if (use_oz) oz.init(b, N, c->chol_slices);
  const TileMaps mapLd = tile_map(Ld, b, 1);
  const TileMaps mapWb = tile_map(Wb, cb, f);
  TileMaps mapPB[4];
  for (int q = 0; q < npb; ++q) mapPB[q] = tile_map(PB[q], b, panel);

  GemmArgs g{};
  g.N = N;
  g.b = b;
  g.cb = cb;
  g.f = f;
  g.A = m->d;
  g.tile_lo = 0;
  g.lpos = m->d_lpos;
  g.flag = flag;

  auto panel_work = [&](int64_t j) {
    const int dj = cyclic_owner(j, j, P, Q);
    if (dj == me) {  // diagonal tile (local)
      for (int s = 0; s < f; ++s) {
        diag128_kernel<<<1, 256, kDiagSmem, cs.p>>>(m->d, 0, m->d_lpos, b, f, m->dinv,
                                                    j * f + s, 0, flag);
        HS_CUDA(cudaGetLastError());
        launch_count(c);
        if (s + 1 < f) {
          GemmArgs gd = g;
          gd.j = j;
          gd.step = s;
          gd.W = m->dinv;
          gd.mode = G_DIAG_TRSM;
          launch_gemm(c, cs.p, gd, f - 1 - s, &mapA, &mapW);
          gd.mode = G_DIAG_UPD;
          const int64_t tt = f - 1 - s;
          launch_gemm(c, cs.p, gd, tt * (tt + 1) / 2, &mapA, &mapA);
        }
      }
    }
    // L_jj and its inverse blocks to every rank
    const int64_t dslot = m->lpos[tri(j, j)];
    c->step = j;
    comm_group(c, true);
    comm_bcast_on(c, dj == me ? m->d + dslot * bb : nullptr, Ld, (size_t)bb, dj, cs.p,
                  LK_BLOCK);
    comm_bcast_on(c, dj == me ? m->dinv + j * f * (int64_t)cb * cb : nullptr, Wb,
                  (size_t)f * cb * cb, dj, cs.p, LK_BLOCK);
    comm_group(c, false);
    // TRSM of the owned panel tiles (in place)
    const int64_t nr = row_off[j + 1] - row_off[j];
    if (nr > 0) {
      for (int cc = 0; cc < f; ++cc) {
        GemmArgs gp = g;
        gp.j = j;
        gp.step = cc;
        gp.list = d_rows + row_off[j];
        gp.X = Ld;
        gp.W = Wb;
        if (cc > 0) {
          gp.mode = G_DIST_PANEL_UPD;
          launch_gemm(c, cs.p, gp, nr * f, &mapA, &mapLd);
        }
        gp.mode = G_DIST_PANEL_TRSM;
        launch_gemm(c, cs.p, gp, nr * f, &mapA, &mapWb);
      }
    }
    // every panel tile from its owner into PB[j & 1] on every rank
    if (j + 1 < N) {
      comm_group(c, true);
      for (int64_t i = j + 1; i < N; ++i) {
        const int own = cyclic_owner(i, j, P, Q);
        const double* send = own == me ? m->d + m->lpos[tri(i, j)] * bb : nullptr;
        comm_bcast_on(c, send, PB[pbi(j)] + (i - j - 1) * bb, (size_t)bb, own, cs.p,
                      LK_BLOCK);
      }
      comm_group(c, false);
      if (use_oz) oz.slice_contig(c, cs.p, PB[pbi(j)], N, j, &flag->status);
    }
  };

  panel_work(0);
  if (dpairs) {
    // the single-GPU pair schedule over the broadcast panels: lookahead
    // updates on U at the panel's priority, the bulk on a low-priority U2
    HS_CUDA(cudaStreamCreateWithPriority(&cs.u2, cudaStreamNonBlocking, lo_pri));
    HS_CUDA(cudaStreamWaitEvent(cs.u2, start));
    HS_CUDA(cudaStreamDestroy(cs.u));
    HS_CUDA(cudaStreamCreateWithPriority(&cs.u, cudaStreamNonBlocking, hi_pri));
    HS_CUDA(cudaStreamWaitEvent(cs.u, start));
    cudaEvent_t rest_done = nullptr;
    for (int64_t j0 = 0, pm = 0; j0 + 1 < N; j0 += 2, ++pm) {
      const int64_t j1 = j0 + 1;
      cudaEvent_t p0 = cs.make();
      HS_CUDA(cudaEventRecord(p0, cs.p));
      HS_CUDA(cudaStreamWaitEvent(cs.u, p0));
      GemmArgs gu = g;
      gu.j = j0;
      gu.mode = G_DIST_UPDATE;
      gu.X = PB[pbi(j0)];
      gu.list = d_pairs + 2 * col_off[j0];
      launch_gemm(c, cs.u, gu, (rest_off[j0] - col_off[j0]) * f * f, &mapPB[pbi(j0)],
                  &mapPB[pbi(j0)]);
      cudaEvent_t ucol = cs.make();
      HS_CUDA(cudaEventRecord(ucol, cs.u));
      HS_CUDA(cudaStreamWaitEvent(cs.p, ucol));
      panel_work(j1);
      if (j1 + 1 >= N) break;
      cudaEvent_t p1 = cs.make();
      HS_CUDA(cudaEventRecord(p1, cs.p));
      HS_CUDA(cudaStreamWaitEvent(cs.u, p1));
      if (rest_done) HS_CUDA(cudaStreamWaitEvent(cs.u, rest_done));  // previous bulk
      GemmArgs gp = g;
      gp.j = j0;
      gp.mode = G_DIST_UPDATE_PAIR;
      const int64_t* o = &pp_off[4 * pm];
      gp.list = d_pairs + 2 * o[0];
      launch_gemm(c, cs.u, gp, (o[1] - o[0]) * f * f, &mapPB[pbi(j0)], &mapPB[pbi(j1)]);
      cudaEvent_t ua = cs.make();
      HS_CUDA(cudaEventRecord(ua, cs.u));
      rest_done = nullptr;
      if (j1 + 2 < N) {
        gp.list = d_pairs + 2 * o[1];
        launch_gemm(c, cs.u, gp, (o[2] - o[1]) * f * f, &mapPB[pbi(j0)], &mapPB[pbi(j1)]);
        cudaEvent_t ub = cs.make();
        HS_CUDA(cudaEventRecord(ub, cs.u));
        if (j1 + 3 < N) {
          HS_CUDA(cudaStreamWaitEvent(cs.u2, ub));
          gp.list = d_pairs + 2 * o[2];
          launch_gemm(c, cs.u2, gp, (o[3] - o[2]) * f * f, &mapPB[pbi(j0)], &mapPB[pbi(j1)]);
          rest_done = cs.make();
          HS_CUDA(cudaEventRecord(rest_done, cs.u2));
        }
      }
      HS_CUDA(cudaStreamWaitEvent(cs.p, ua));
      panel_work(j1 + 1);
    }
  }
  for (int64_t j = 0; j < N && !dpairs; ++j) {
    cudaEvent_t pdone = cs.make();
    HS_CUDA(cudaEventRecord(pdone, cs.p));
    if (j + 1 >= N) break;
    HS_CUDA(cudaStreamWaitEvent(cs_u, pdone));
    GemmArgs gu = g;
    gu.j = j;
    gu.mode = G_DIST_UPDATE;
    gu.X = PB[j & 1];
    gu.list = d_pairs + 2 * col_off[j];
    if (use_oz)
      oz.update_list(c, cs_u, m->d, m->d_lpos, j, gu.list, rest_off[j] - col_off[j],
                     &flag->status);
    else
      launch_gemm(c, cs_u, gu, (rest_off[j] - col_off[j]) * f * f, &mapPB[j & 1],
                  &mapPB[j & 1]);
    cudaEvent_t ucol = cs.make();
    HS_CUDA(cudaEventRecord(ucol, cs_u));
    HS_CUDA(cudaStreamWaitEvent(cs.p, ucol));
    gu.list = d_pairs + 2 * rest_off[j];
    if (use_oz)
      oz.update_list(c, cs_u, m->d, m->d_lpos, j, gu.list, col_off[j + 1] - rest_off[j],
                     &flag->status);
    else
      launch_gemm(c, cs_u, gu, (col_off[j + 1] - rest_off[j]) * f * f, &mapPB[j & 1],
                  &mapPB[j & 1]);
    panel_work(j + 1);
  }
  cudaEvent_t pend = cs.make(), uend = cs.make();
  HS_CUDA(cudaEventRecord(pend, cs.p));
  HS_CUDA(cudaEventRecord(uend, cs.u));
  HS_CUDA(cudaStreamWaitEvent(c->stream, pend));
  HS_CUDA(cudaStreamWaitEvent(c->stream, uend));
  if (cs.u2) {
    cudaEvent_t u2end = cs.make();
    HS_CUDA(cudaEventRecord(u2end, cs.u2));
    HS_CUDA(cudaStreamWaitEvent(c->stream, u2end));
  }
  check_finite_kernel<<<4 * 148, 256, 0, c->stream>>>(
      m->d, 0, m->d_owned, (int64_t)m->local_tiles(), b, flag);
  HS_CUDA(cudaGetLastError());
  launch_count(c);
  // agree on the outcome: the earliest failing column wins
  CholFlag h{};
  HS_CUDA(cudaMemcpyAsync(&h, flag, sizeof(h), cudaMemcpyDeviceToHost, c->stream));
  HS_CUDA(cudaStreamSynchronize(c->stream));
  c->step = -1;
  h = agree_on_flag(c, h, d_status);
  throw_flag(h);
  m->has_inv = true;
}

// inverses of all diagonal cb-blocks of an (uploaded) factor; singular check
static void ensure_inverses(hs_ctx* c, hs_matrix* m) {
  if (m->has_inv) return;
  const int b = (int)m->b;
  const int cb = compute_block(b), f = b / cb;
  const int64_t N = (int64_t)m->N;
  set_tile_kernel_attrs(b);
  alloc_inverses(m);
  CholFlag* flag = static_cast<CholFlag*>(ctx_scratch(c)) + 2;
  HS_CUDA(cudaMemsetAsync(flag, 0, sizeof(CholFlag), c->stream));
  if (c->world > 1) {
    // block-cyclic factor: each rank inverts the diagonal tiles it owns
    // (the ones its substitution steps use), and all agree on the outcome
    HS_REQUIRE(dmma_ok(b) && m->layout == 1, HS_ERR_CONFIG,
               "multi-rank triangular solves need a block-cyclic factor with b % 128 == 0");
    for (int64_t j = 0; j < N; ++j)
      if (cyclic_owner(j, j, m->P, m->Q) == c->rank) {
        diag128_kernel<<<(unsigned)f, 256, kDiagSmem, c->stream>>>(
            m->d, 0, m->d_lpos, b, f, m->dinv, j * f, 1, flag);
        HS_CUDA(cudaGetLastError());
        launch_count(c);
      }
    CholFlag h{};
    HS_CUDA(cudaMemcpyAsync(&h, flag, sizeof(h), cudaMemcpyDeviceToHost, c->stream));
    HS_CUDA(cudaStreamSynchronize(c->stream));
    c->step = -1;
    h = agree_on_flag(c, h, reinterpret_cast<int64_t*>(flag));
    throw_flag(h);
    m->has_inv = true;
    return;
  }
  if (dmma_ok(b)) {
    diag128_kernel<<<(unsigned)(N * f), 256, kDiagSmem, c->stream>>>(
        m->d, m->tile_lo, m->d_lpos, b, f, m->dinv, 0, 1, flag);
  } else {
    trtri_tile_kernel<<<(unsigned)N, 256, trtri_smem(b), c->stream>>>(
        m->d, m->tile_lo, m->dinv, b, flag, 0);
  }
  HS_CUDA(cudaGetLastError());
  launch_count(c);
  CholFlag h{};
  HS_CUDA(cudaMemcpyAsync(&h, flag, sizeof(h), cudaMemcpyDeviceToHost, c->stream));
  HS_CUDA(cudaStreamSynchronize(c->stream));
  throw_flag(h);
  m->has_inv = true;
}

// Multi-rank substitution over the 2D block-cyclic factor (SURVEY §8e:
// pipelined over tile rows, b-double blocks on the wire). Every rank holds
// the full vector v on entry and exit. Step i (forward i = 0..N-1, backward
// i = N-1..0):
//   all-gather the b-double slice i of each rank's partial-update vector w
//     (w_k accumulates -L_ki y_i over the rank's own tiles);
//   owner(i, i): v_i = W_i (v_i + sum_r w_i^(r)) with the stored inverse
//     blocks (rank-order sum: identical on every run);
//   broadcast v_i from owner(i, i);
//   every rank: w_k -= L_ki v_i (forward, owned tiles below i) or
//     w_k -= L_ik^T v_i (backward, owned tiles left of i).
// The reference runs both substitutions on the one executor holding the
// factor (cholesky_solver.cpp:287-309); with the factor spread over ranks
// the steps are pipelined over tile rows instead and only b-double blocks
// move, never a tile.
// The substitution kernels stage 2b doubles (+ the diagonal tile's share)
// in shared memory: b <= 2048. Checked before any factorization that is
// followed by a solve, so an unsupported b fails before A is overwritten.
static void require_trsv_block(size_t b) {
  HS_REQUIRE(b <= 2048, HS_ERR_CONFIG,
             "block size " + std::to_string(b) +
                 " unsupported in the triangular solves (b <= 2048)");
}

static void trsv_run_dist(hs_ctx* c, hs_matrix* m, double* v, bool upper) {
  HS_REQUIRE(m->layout == 1, HS_ERR_CONFIG,
             "multi-rank triangular solves need a block-cyclic factor");
  require_trsv_block(m->b);
  ensure_inverses(c, m);
  const int b = (int)m->b;
  const int cb = compute_block(b), f = b / cb;
  const int64_t N = (int64_t)m->N;
  const int P = m->P, Q = m->Q, me = c->rank, G = c->world;
  const size_t dsm = (2 * (size_t)b + (trsv_staged(b, cb, f) ? trsv_staged_doubles(cb, f) : 0)) *
                         sizeof(double),
               usm = (size_t)b * sizeof(double);
  if (dsm > 48 * 1024)
    HS_CUDA(cudaFuncSetAttribute(trsv_diag_kernel,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dsm));
  // per step, the owned tiles this rank applies v_i through
  std::vector<int32_t> list;
  std::vector<int64_t> off(N + 1, 0);
  for (int64_t s = 0; s < N; ++s) {
    const int64_t i = upper ? N - 1 - s : s;
    off[s] = (int64_t)list.size();
    if (upper) {
      for (int64_t k = 0; k < i; ++k)
        if (cyclic_owner(i, k, P, Q) == me) list.push_back((int32_t)k);
    } else {
      for (int64_t k = i + 1; k < N; ++k)
        if (cyclic_owner(k, i, P, Q) == me) list.push_back((int32_t)k);
    }
  }
  off[N] = (int64_t)list.size();
  const size_t sz[3] = {(size_t)N * b * sizeof(double), (size_t)G * b * sizeof(double),
                        std::max<size_t>(list.size(), 1) * sizeof(int32_t)};
  void* ws[3];
  ctx_workspace(c, 2, sz, 3, ws);  // persistent across calls
  double* w = static_cast<double*>(ws[0]);
  double* gath = static_cast<double*>(ws[1]);
  int32_t* d_list = static_cast<int32_t*>(ws[2]);
  HS_CUDA(cudaMemcpyAsync(d_list, list.data(), list.size() * sizeof(int32_t),
                          cudaMemcpyHostToDevice, c->stream));
  HS_CUDA(cudaMemsetAsync(w, 0, (size_t)N * b * sizeof(double), c->stream));
  for (int64_t s = 0; s < N; ++s) {
    const int64_t i = upper ? N - 1 - s : s;
    const int root = cyclic_owner(i, i, P, Q);
    c->step = i;
    // nobody has touched w_i before the first step
    const bool gather = s > 0;
    if (gather) comm_allgather(c, w + i * b, gath, (size_t)b, LK_SUBVECTOR);
    if (root == me) {
      HS_CUDA(launch_pdl_cluster(trsv_diag_kernel, dim3(TRSV_CLUSTER), dim3(TRSV_DIAG_THREADS),
                         TRSV_CLUSTER, dsm,
                         c->stream, (const double*)m->d, (int64_t)0,
                         (const int64_t*)m->d_lpos, (const double*)m->dinv, v,
                         gather ? (const double*)gath : nullptr, G, b, cb, f, i,
                         upper ? 1 : 0));
      launch_count(c);
    }
    comm_bcast_on(c, v + i * b, v + i * b, (size_t)b, root, c->stream, LK_SUBVECTOR);
    const int64_t nk = off[s + 1] - off[s];
    if (nk > 0) {
      const int mode = trsv_mode(b, upper, nk);
      HS_CUDA(launch_trsv_update(mode, dim3(trsv_chunks(b, mode), (unsigned)nk), usm,
                         c->stream, (const double*)m->d, (int64_t)0,
                         (const int64_t*)m->d_lpos, (const int32_t*)(d_list + off[s]),
                         (const double*)v, w, b, i, mode));
      launch_count(c);
    }
  }
  c->step = -1;
  HS_CUDA(cudaStreamSynchronize(c->stream));
}

static void trsv_run(hs_ctx* c, hs_matrix* m, double* v, bool upper) {
  if (c->world > 1) return trsv_run_dist(c, m, v, upper);
  ensure_inverses(c, m);
  const int b = (int)m->b;
  const int cb = compute_block(b), f = b / cb;
  require_trsv_block(m->b);
  const int64_t N = (int64_t)m->N;
  const size_t dsm = (2 * (size_t)b + (trsv_staged(b, cb, f) ? trsv_staged_doubles(cb, f) : 0)) *
                         sizeof(double),
               usm = (size_t)b * sizeof(double);
  if (dsm > 48 * 1024)
    HS_CUDA(cudaFuncSetAttribute(trsv_diag_kernel,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dsm));
  for (int64_t s = 0; s < N; ++s) {
    const int64_t i = upper ? N - 1 - s : s;
    HS_CUDA(launch_pdl_cluster(trsv_diag_kernel, dim3(TRSV_CLUSTER), dim3(TRSV_DIAG_THREADS),
                         TRSV_CLUSTER, dsm,
                       c->stream, (const double*)m->d, m->tile_lo, (const int64_t*)nullptr,
                       (const double*)m->dinv, v, (const double*)nullptr, 1, b, cb, f, i,
                       upper ? 1 : 0));
    launch_count(c);
    const int64_t nk = upper ? i : N - 1 - i;
    if (nk > 0) {
      const int mode = trsv_mode(b, upper, nk);
      HS_CUDA(launch_trsv_update(mode, dim3(trsv_chunks(b, mode), (unsigned)nk), usm,
                         c->stream, (const double*)m->d, m->tile_lo, (const int64_t*)nullptr,
                         (const int32_t*)nullptr, (const double*)v, v, b, i, mode));
      launch_count(c);
    }
  }
  HS_CUDA(cudaStreamSynchronize(c->stream));
}

// ---- iterative refinement helpers (hs_solve_spd_refine) -------------------
// y = a + alpha z (element-wise; y may alias a or z)
__global__ void refine_axpy_kernel(double* y, const double* a, double alpha, const double* z,
                                   int64_t n) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x)
    y[k] = fma(alpha, z[k], a[k]);
}
// *out = u . v, one CTA in a fixed order (deterministic)
__global__ void __launch_bounds__(1024) refine_dot_kernel(const double* u, const double* v,
                                                          int64_t n, double* out) {
  __shared__ double red[32];
  double s = 0.0;
  for (int64_t k = threadIdx.x; k < n; k += blockDim.x) s = fma(u[k], v[k], s);
  for (int off = 16; off; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    s = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
    for (int off = 16; off; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
    if (threadIdx.x == 0) *out = s;
  }
}
// *out = ||v||_2, one CTA in a fixed order (deterministic)
__global__ void __launch_bounds__(1024) refine_norm2_kernel(const double* v, int64_t n,
                                                            double* out) {
  __shared__ double red[32];
  double s = 0.0;
  for (int64_t k = threadIdx.x; k < n; k += blockDim.x) s = fma(v[k], v[k], s);
  for (int off = 16; off; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    s = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
    for (int off = 16; off; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
    if (threadIdx.x == 0) *out = sqrt(s);
  }
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
  require_trsv_block(a->b);  // before the factorization overwrites A
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

hs_status hs_solve_spd_refine(hs_ctx* c, const hs_matrix* a, hs_matrix* w,
                              const double* d_rhs, double* d_x, int slices, int max_iters,
                              double tol, hs_refine_stats* st) {
  HS_API_BEGIN
  HS_REQUIRE(c && a && w && d_rhs && d_x, HS_ERR_CONFIG, "null pointer");
  HS_REQUIRE(a->layout == w->layout && (c->world == 1 || a->layout == 1), HS_ERR_CONFIG,
             "multi-rank hs_solve_spd_refine needs block-cyclic matrices");
  HS_REQUIRE(a->n == w->n && a->b == w->b, HS_ERR_CONFIG, "work matrix shape differs from a");
  HS_REQUIRE(slices >= 0 && slices <= 8 && max_iters >= 0 && tol >= 0.0, HS_ERR_CONFIG,
             "slices in [0, 8], max_iters >= 0, tol >= 0");
  require_trsv_block(a->b);
  HS_CUDA(cudaSetDevice(c->device));
  hs_refine_stats s{};
  s.slices = slices;
  const auto t0 = std::chrono::steady_clock::now();
  hs_status r = hs_matrix_copy(w, a);
  if (r != HS_OK) throw Failure{r, hs_last_error()};
  {
    const int saved = c->chol_slices;
    c->chol_slices = slices;
    try {
      potrf_run(c, w);
    } catch (...) {
      c->chol_slices = saved;
      throw;
    }
    c->chol_slices = saved;
  }
  s.factor_ms = ms_since(t0);
  const auto t1 = std::chrono::steady_clock::now();
  const int64_t pn = (int64_t)a->N * (int64_t)a->b;
  // residual / correction; PCG: z, p, q; then a scalar slot
  double* res = ctx_vec(c, 3, 4 * (size_t)pn + 1);
  double* zv = res + pn;
  double* pv = zv + pn;
  double* qv = pv + pn;
  double* nrm = qv + pn;
  auto norm2 = [&](const double* v) {
    refine_norm2_kernel<<<1, 1024, 0, c->stream>>>(v, pn, nrm);
    HS_CUDA(cudaGetLastError());
    launch_count(c);
    double h = 0.0;
    HS_CUDA(cudaMemcpyAsync(&h, nrm, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    HS_CUDA(cudaStreamSynchronize(c->stream));
    return h;
  };
  const unsigned vg = (unsigned)std::min<int64_t>(4 * 148, ceil_div(pn, 256));
  HS_CUDA(cudaMemcpyAsync(d_x, d_rhs, pn * sizeof(double), cudaMemcpyDeviceToDevice,
                          c->stream));
  trsv_run(c, w, d_x, false);
  trsv_run(c, w, d_x, true);
  const double rhs_norm = norm2(d_rhs);
  double prev = -1.0;
  // HS_REFINE_PCG=1: conjugate gradients preconditioned with the factor
  // (x0 = M^-1 rhs; each step one more SYMV for q = A p, and the true
  // residual rhs - A x in place of the recursive one)
  static const bool pcg = [] {
    const char* e = getenv("HS_REFINE_PCG");
    return e && atoi(e) != 0;
  }();
  auto dot = [&](const double* u, const double* v) {
    refine_dot_kernel<<<1, 1024, 0, c->stream>>>(u, v, pn, nrm);
    HS_CUDA(cudaGetLastError());
    launch_count(c);
    double h = 0.0;
    HS_CUDA(cudaMemcpyAsync(&h, nrm, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    HS_CUDA(cudaStreamSynchronize(c->stream));
    return h;
  };
  auto launch_axpy = [&](double* y, const double* a0, double alpha, const double* z) {
    refine_axpy_kernel<<<vg, 256, 0, c->stream>>>(y, a0, alpha, z, pn);
    HS_CUDA(cudaGetLastError());
    launch_count(c);
  };
  if (pcg) {
    double rz = 0.0;
    for (int it = 0;; ++it) {
      symv_full(c, a, d_x, res);
      launch_axpy(res, d_rhs, -1.0, res);  // r = rhs - A x
      const double rn = norm2(res);
      s.rel_residual = rhs_norm > 0.0 ? rn / rhs_norm : rn;
      if (!(s.rel_residual > tol) || it == max_iters || (prev >= 0.0 && rn > 0.5 * prev)) break;
      prev = rn;
      HS_CUDA(cudaMemcpyAsync(zv, res, pn * sizeof(double), cudaMemcpyDeviceToDevice,
                              c->stream));
      trsv_run(c, w, zv, false);
      trsv_run(c, w, zv, true);  // z = M^-1 r
      const double rz_new = dot(res, zv);
      if (it == 0)
        HS_CUDA(cudaMemcpyAsync(pv, zv, pn * sizeof(double), cudaMemcpyDeviceToDevice,
                                c->stream));
      else
        launch_axpy(pv, zv, rz_new / rz, pv);  // p = z + beta p
      rz = rz_new;
      symv_full(c, a, pv, qv);  // q = A p
      const double pq = dot(pv, qv);
      if (!(pq > 0.0)) break;
      launch_axpy(d_x, d_x, rz / pq, pv);  // x += alpha p
      s.iterations = it + 1;
    }
    HS_CUDA(cudaStreamSynchronize(c->stream));
    s.solve_ms = ms_since(t1);
    s.wall_ms = ms_since(t0);
    if (st) *st = s;
    return HS_OK;
  }
  for (int it = 0;; ++it) {
    symv_full(c, a, d_x, res);  // res = A x (FP64, the unmodified matrix; every rank)
    refine_axpy_kernel<<<vg, 256, 0, c->stream>>>(res, d_rhs, -1.0, res, pn);  // rhs - A x
    HS_CUDA(cudaGetLastError());
    launch_count(c);
    const double rn = norm2(res);
    s.rel_residual = rhs_norm > 0.0 ? rn / rhs_norm : rn;
    // done: below tol, out of steps, or stagnated -- the last step did not
    // halve the residual (FP64 rounding floor of rhs - A x reached)
    if (!(s.rel_residual > tol) || it == max_iters || (prev >= 0.0 && rn > 0.5 * prev)) break;
    prev = rn;
    trsv_run(c, w, res, false);
    trsv_run(c, w, res, true);
    refine_axpy_kernel<<<vg, 256, 0, c->stream>>>(d_x, d_x, 1.0, res, pn);  // x += d
    HS_CUDA(cudaGetLastError());
    launch_count(c);
    s.iterations = it + 1;
  }
  HS_CUDA(cudaStreamSynchronize(c->stream));
  s.solve_ms = ms_since(t1);
  s.wall_ms = ms_since(t0);
  if (st) *st = s;
  HS_API_END
}

hs_status hs_factorize_host(hs_ctx* c, size_t n, size_t b, double* a_packed,
                            hs_chol_stats* st) {
  HS_API_BEGIN
  HS_REQUIRE(c && a_packed, HS_ERR_CONFIG, "null pointer");
  HS_CUDA(cudaSetDevice(c->device));
  hs_matrix* m = cached_matrix(c, 0, n, b);
  hs_status s = HS_OK;
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
  require_trsv_block(b);
  HS_CUDA(cudaSetDevice(c->device));
  hs_matrix* m = cached_matrix(c, 0, n, b);
  hs_matrix* orig = cached_matrix(c, 1, n, b);
  hs_status s = HS_OK;
  const size_t pn = (size_t)ceil_div(n, b) * b;
  double* d_rhs = ctx_vec(c, 0, pn);
  double* d_x = ctx_vec(c, 1, pn);
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
  // the context's cached device matrix and vector (kept across calls)
  hs_matrix* m = cached_matrix(c, 0, n, b);
  const hs_status s = hs_matrix_upload(m, l);
  if (s != HS_OK) throw Failure{s, hs_last_error()};
  const size_t pn = (size_t)ceil_div(n, b) * b;
  double* d_v = ctx_vec(c, 2, pn);
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
  // the context's cached device matrix and vector (kept across calls)
  hs_matrix* m = cached_matrix(c, 0, n, b);
  const hs_status s = hs_matrix_upload(m, l);
  if (s != HS_OK) throw Failure{s, hs_last_error()};
  const size_t pn = (size_t)ceil_div(n, b) * b;
  double* d_v = ctx_vec(c, 2, pn);
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
  set_simt_tile_attrs((int)b);
  CholFlag* flag = static_cast<CholFlag*>(ctx_scratch(c)) + 3;
  HS_CUDA(cudaMemsetAsync(flag, 0, sizeof(CholFlag), c->stream));
  potrf_tile_kernel<<<(unsigned)count, 256, potrf_smem((int)b), c->stream>>>(
      d_tiles, (int64_t)(b * b), (int)b, flag, -1);
  HS_CUDA(cudaGetLastError());
  launch_count(c);
  CholFlag h{};
  HS_CUDA(cudaMemcpyAsync(&h, flag, sizeof(h), cudaMemcpyDeviceToHost, c->stream));
  HS_CUDA(cudaStreamSynchronize(c->stream));
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
  g.cb = compute_block((int)b);
  g.f = (int)b / g.cb;
  g.C = d_c;
  g.P = d_p;
  g.Q = d_q;
  g.lower_only = lower_only;
  const int64_t items = (int64_t)count * g.f * g.f;
  if (dmma_ok((int)b)) {
    TileMaps mp = tile_map(d_p, (int)b, (int64_t)count);
    TileMaps mq = tile_map(d_q, (int)b, (int64_t)count);
    launch_gemm(c, c->stream, g, items, &mp, &mq);
  } else {
    launch_gemm(c, c->stream, g, items, nullptr, nullptr);
  }
  HS_CUDA(cudaStreamSynchronize(c->stream));
  HS_API_END
}

}  // extern "C"
