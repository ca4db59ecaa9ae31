// Single-block and block-row-range kernels behind the reference's kernel API
// (include/hsolve/block_kernels.hpp, reference block_kernels.hpp:16-74):
// TRSM of one tile, the four single-block GEMV / triangular-solve kernels of
// the substitutions, per-row dots and the axpy / xpay / sub range updates.
// Every output element is one sequential chain in the reference's order with
// separately rounded multiply and add (__dmul_rn / __dadd_rn / __dsub_rn,
// no FMA contraction), so these reproduce block_kernels.cpp bitwise; they
// are the kernel-level drop-in, not the solvers' hot path (which runs the
// tiled DMMA / TMA kernels of hs_chol.cu and hs_cg.cu).
#include <cmath>
#include <string>
#include <vector>

#include "hs_internal.h"

namespace hs {

// X L^T = B in place, per row of X (block_kernels.cpp:23-37): thread r owns
// row r; column c needs the row's columns < c only.
__global__ void trsm_rows_kernel(double* x, const double* l, int b, int64_t stride_x,
                                 int64_t stride_l) {
  double* xt = x + blockIdx.y * stride_x;
  const double* lt = l + blockIdx.y * stride_l;
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < b; r += gridDim.x * blockDim.x) {
    double* xr = xt + (int64_t)r * b;
    for (int c = 0; c < b; ++c) {
      double acc = xr[c];
      for (int k = 0; k < c; ++k) acc = __dsub_rn(acc, __dmul_rn(xr[k], lt[(int64_t)c * b + k]));
      xr[c] = __ddiv_rn(acc, lt[(int64_t)c * b + c]);
    }
  }
}

// c -= p q^T (lower_only: col <= r) per element, k ascending from 0
// (block_kernels.cpp:39-57)
__global__ void gemm_exact_kernel(double* c, const double* p, const double* q, int b,
                                  int lower_only) {
  const int64_t bb = (int64_t)b * b;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < bb;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(e / b), col = (int)(e - (int64_t)r * b);
    if (lower_only && col > r) continue;
    double acc = 0.0;
    for (int k = 0; k < b; ++k)
      acc = __dadd_rn(acc, __dmul_rn(p[(int64_t)r * b + k], q[(int64_t)col * b + k]));
    c[e] = __dsub_rn(c[e], acc);
  }
}

// potf_block (block_kernels.cpp:9-21): thread p owns row p and runs the
// reference's loops over it; element (p, q) needs row q finished, which its
// owner publishes through a shared-memory flag (rows complete in order, so
// the rows pipeline). The first failing pivot row wins, as in the
// reference's row order.
__global__ void potf_exact_kernel(double* d, int b, int* bad) {
  extern __shared__ int row_done[];
  for (int r = threadIdx.x; r < b; r += blockDim.x) row_done[r] = 0;
  __syncthreads();
  const int p = threadIdx.x;
  if (p < b) {
    double* dp = d + (int64_t)p * b;
    for (int q = 0; q < p; ++q) {
      while (atomicAdd(&row_done[q], 0) == 0) {
      }
      __threadfence_block();
      const double* dq = d + (int64_t)q * b;
      double acc = dp[q];
      for (int k = 0; k < q; ++k) acc = __dsub_rn(acc, __dmul_rn(dp[k], dq[k]));
      dp[q] = __ddiv_rn(acc, dq[q]);
    }
    double acc = dp[p];
    for (int k = 0; k < p; ++k) acc = __dsub_rn(acc, __dmul_rn(dp[k], dp[k]));
    if (!(acc > 0.0)) atomicMin(bad, p);
    dp[p] = __dsqrt_rn(acc);
    __threadfence_block();
    atomicExch(&row_done[p], 1);
  }
}

// symv_row (block_kernels.cpp:59-95) for rows [r0, r1) of the padded
// system: one thread per output row, ascending j then c, unfused
__global__ void symv_exact_kernel(const double* a, const double* x, double* y, int64_t rows,
                                  int b, int64_t r0, int64_t r1) {
  for (int64_t pr = r0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; pr < r1;
       pr += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = pr / b;
    const int r = (int)(pr - i * b);
    double acc = 0.0;
    for (int64_t j = 0; j < rows; ++j) {
      const double* xj = x + j * b;
      if (j <= i) {
        const double* blk = a + tri(i, j) * b * b;
        for (int c = 0; c < b; ++c) {
          const double v = (j < i || c <= r) ? blk[(int64_t)r * b + c] : blk[(int64_t)c * b + r];
          acc = __dadd_rn(acc, __dmul_rn(v, xj[c]));
        }
      } else {
        const double* blk = a + tri(j, i) * b * b;
        for (int c = 0; c < b; ++c) acc = __dadd_rn(acc, __dmul_rn(blk[(int64_t)c * b + r], xj[c]));
      }
    }
    y[pr] = acc;
  }
}

// the diagonal check of trsm_block / lower_solve: first zero or NaN index
__global__ void diag_check_kernel(const double* l, int b, int64_t* bad) {
  for (int c = threadIdx.x; c < b; c += blockDim.x) {
    const double d = l[(int64_t)c * b + c];
    if (d == 0.0 || isnan(d)) atomicMin(reinterpret_cast<unsigned long long*>(bad),
                                        (unsigned long long)c);
  }
}

// y -= M x / y -= M^T x (block_kernels.cpp:154-169)
__global__ void gemv_sub_kernel(const double* m, const double* x, double* y, int b, int trans) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < b; r += gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (int c = 0; c < b; ++c) {
      const double mv = trans ? m[(int64_t)c * b + r] : m[(int64_t)r * b + c];
      acc = __dadd_rn(acc, __dmul_rn(mv, x[c]));
    }
    y[r] = __dsub_rn(y[r], acc);
  }
}

// lower_solve / lower_transpose_solve (block_kernels.cpp:171-189): element r
// needs every earlier one, so a single thread runs the reference's loops
__global__ void lower_solve_kernel(const double* l, double* y, int b, int trans) {
  if (threadIdx.x != 0) return;
  if (!trans) {
    for (int r = 0; r < b; ++r) {
      double acc = y[r];
      for (int c = 0; c < r; ++c) acc = __dsub_rn(acc, __dmul_rn(l[(int64_t)r * b + c], y[c]));
      y[r] = __ddiv_rn(acc, l[(int64_t)r * b + r]);
    }
  } else {
    for (int rr = b - 1; rr >= 0; --rr) {
      double acc = y[rr];
      for (int c = rr + 1; c < b; ++c)
        acc = __dsub_rn(acc, __dmul_rn(l[(int64_t)c * b + rr], y[c]));
      y[rr] = __ddiv_rn(acc, l[(int64_t)rr * b + rr]);
    }
  }
}

// block-row range ops over padded vectors (block_kernels.cpp:102-152)
__global__ void range_kernel(int op, double* out, const double* u, const double* v, double alpha,
                             int64_t lo, int64_t hi, int b) {
  const int64_t n = (hi - lo) * b;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < (op == 0 ? hi - lo : n);
       k += (int64_t)gridDim.x * blockDim.x) {
    if (op == 0) {  // row_dot of row lo + k into out[lo + k]
      const int64_t o = (lo + k) * b;
      double acc = 0.0;
      for (int c = 0; c < b; ++c) acc = __dadd_rn(acc, __dmul_rn(u[o + c], v[o + c]));
      out[lo + k] = acc;
    } else {
      const int64_t e = lo * b + k;
      if (op == 1) out[e] = __dadd_rn(out[e], __dmul_rn(alpha, u[e]));       // axpy
      else if (op == 2) out[e] = __dadd_rn(u[e], __dmul_rn(alpha, out[e]));  // xpay
      else out[e] = __dsub_rn(u[e], v[e]);                                   // sub
    }
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

static int64_t first_singular(hs_ctx* c, const double* l, int b) {
  int64_t* bad = static_cast<int64_t*>(ctx_scratch(c)) + 16;
  const int64_t none = INT64_MAX;
  HS_CUDA(cudaMemcpyAsync(bad, &none, sizeof(none), cudaMemcpyHostToDevice, c->stream));
  diag_check_kernel<<<1, 256, 0, c->stream>>>(l, b, bad);
  HS_CUDA(cudaGetLastError());
  launch_count(c);
  int64_t h = none;
  HS_CUDA(cudaMemcpyAsync(&h, bad, sizeof(h), cudaMemcpyDeviceToHost, c->stream));
  HS_CUDA(cudaStreamSynchronize(c->stream));
  return h == none ? -1 : h;
}

extern "C" {

hs_status hs_trsm_tiles(hs_ctx* c, double* d_x, const double* d_l, size_t b, size_t count) {
  HS_API_BEGIN
  HS_REQUIRE(c && d_x && d_l && b > 0, HS_ERR_CONFIG, "bad trsm request");
  HS_CUDA(cudaSetDevice(c->device));
  const int64_t bb = (int64_t)b * b;
  for (size_t t = 0; t < count; ++t) {
    const int64_t bad = first_singular(c, d_l + t * bb, (int)b);
    if (bad >= 0) {
      throw Failure{HS_ERR_SINGULAR_BLOCK,
                    "triangular block has zero or NaN diagonal at index " + std::to_string(bad),
                    -1, bad};
    }
  }
  if (count) {
    const dim3 grid((unsigned)ceil_div((int64_t)b, 128), (unsigned)count);
    trsm_rows_kernel<<<grid, 128, 0, c->stream>>>(d_x, d_l, (int)b, bb, bb);
    HS_CUDA(cudaGetLastError());
    launch_count(c);
  }
  HS_CUDA(cudaStreamSynchronize(c->stream));
  HS_API_END
}

hs_status hs_block_exact(hs_ctx* c, int op, double* d_c, const double* d_p, const double* d_q,
                         size_t b, int64_t* bad_pivot) {
  HS_API_BEGIN
  HS_REQUIRE(c && d_c && b > 0 && op >= 0 && op <= 2, HS_ERR_CONFIG, "bad block op");
  HS_CUDA(cudaSetDevice(c->device));
  if (op == 0) {
    HS_REQUIRE(b <= 1024, HS_ERR_CONFIG, "potf_block: b <= 1024 on the device");
    int* bad = static_cast<int*>(ctx_scratch(c)) + 48;
    const int none = 0x7fffffff;
    HS_CUDA(cudaMemcpyAsync(bad, &none, sizeof(int), cudaMemcpyHostToDevice, c->stream));
    potf_exact_kernel<<<1, (unsigned)((b + 31) / 32 * 32), b * sizeof(int), c->stream>>>(
        d_c, (int)b, bad);
    HS_CUDA(cudaGetLastError());
    launch_count(c);
    int h = none;
    HS_CUDA(cudaMemcpyAsync(&h, bad, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    HS_CUDA(cudaStreamSynchronize(c->stream));
    if (bad_pivot) *bad_pivot = h == none ? -1 : h;
    if (h != none)
      throw Failure{HS_ERR_NOT_SPD,
                    "matrix is not positive definite (block row -1, pivot " +
                        std::to_string(h) + ")",
                    -1, h};
    return HS_OK;
  }
  HS_REQUIRE(d_p && d_q, HS_ERR_CONFIG, "null operand");
  gemm_exact_kernel<<<296, 256, 0, c->stream>>>(d_c, d_p, d_q, (int)b, op == 2 ? 1 : 0);
  HS_CUDA(cudaGetLastError());
  launch_count(c);
  HS_CUDA(cudaStreamSynchronize(c->stream));
  HS_API_END
}

hs_status hs_symv_exact(hs_ctx* c, const double* d_a, const double* d_x, double* d_y, size_t n,
                        size_t b, size_t lo, size_t hi) {
  HS_API_BEGIN
  HS_REQUIRE(c && d_a && d_x && d_y && b > 0 && lo <= hi, HS_ERR_CONFIG, "bad symv request");
  HS_CUDA(cudaSetDevice(c->device));
  const int64_t rows = ceil_div((int64_t)n, (int64_t)b);
  HS_REQUIRE((int64_t)hi <= rows, HS_ERR_CONFIG, "block-row range out of range");
  if (hi > lo) {
    symv_exact_kernel<<<296, 128, 0, c->stream>>>(d_a, d_x, d_y, rows, (int)b,
                                                  (int64_t)lo * b, (int64_t)hi * b);
    HS_CUDA(cudaGetLastError());
    launch_count(c);
  }
  HS_CUDA(cudaStreamSynchronize(c->stream));
  HS_API_END
}

hs_status hs_block_vec_op(hs_ctx* c, int op, const double* d_m, const double* d_x, double* d_y,
                          size_t b) {
  HS_API_BEGIN
  HS_REQUIRE(c && d_m && d_y && b > 0 && op >= 0 && op <= 3, HS_ERR_CONFIG,
             "bad block vector op");
  HS_CUDA(cudaSetDevice(c->device));
  if (op <= 1) {
    HS_REQUIRE(d_x, HS_ERR_CONFIG, "null vector");
    gemv_sub_kernel<<<(unsigned)ceil_div((int64_t)b, 128), 128, 0, c->stream>>>(d_m, d_x, d_y,
                                                                              (int)b, op);
  } else {
    const int64_t bad = first_singular(c, d_m, (int)b);
    if (bad >= 0) {
      // the reference checks row by row and throws at the first bad row it
      // reaches: ascending for lower_solve, descending for the transpose
      int64_t at = bad;
      if (op == 3) {
        std::vector<double> diag(b);
        for (size_t r = 0; r < b; ++r)
          HS_CUDA(cudaMemcpy(&diag[r], d_m + r * b + r, sizeof(double), cudaMemcpyDeviceToHost));
        for (size_t r = b; r-- > 0;)
          if (diag[r] == 0.0 || std::isnan(diag[r])) {
            at = (int64_t)r;
            break;
          }
      }
      throw Failure{HS_ERR_SINGULAR_BLOCK,
                    "triangular block has zero or NaN diagonal at index " + std::to_string(at),
                    -1, at};
    }
    lower_solve_kernel<<<1, 32, 0, c->stream>>>(d_m, d_y, (int)b, op - 2);
  }
  HS_CUDA(cudaGetLastError());
  launch_count(c);
  HS_CUDA(cudaStreamSynchronize(c->stream));
  HS_API_END
}

hs_status hs_range_op(hs_ctx* c, int op, double* d_out, const double* d_u, const double* d_v,
                      double alpha, size_t lo, size_t hi, size_t b) {
  HS_API_BEGIN
  HS_REQUIRE(c && d_out && b > 0 && lo <= hi && op >= 0 && op <= 3, HS_ERR_CONFIG,
             "bad range op");
  HS_CUDA(cudaSetDevice(c->device));
  if (hi > lo) {
    range_kernel<<<296, 256, 0, c->stream>>>(op, d_out, d_u, d_v, alpha, (int64_t)lo,
                                             (int64_t)hi, (int)b);
    HS_CUDA(cudaGetLastError());
    launch_count(c);
  }
  HS_CUDA(cudaStreamSynchronize(c->stream));
  HS_API_END
}

}  // extern "C"
