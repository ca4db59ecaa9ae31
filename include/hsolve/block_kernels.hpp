// Kernel-level drop-in for the reference's hsolve::kernels (reference
// include/hsolve/block_kernels.hpp:16-74): the same 17 functions and
// signatures on host buffers. Each call runs on the GPU of the process's
// default context (device 0): the operands are copied in, one sm_100a kernel
// computes, the result is copied back. Every output element is one sequential
// chain in the reference's order with separately rounded multiply and add
// (no FMA contraction), so results match the reference bitwise; potf_block
// pipelines its rows (thread per row, b <= 1024).
//
// These are per-block utilities for callers that assemble their own solvers
// from the reference's kernels; the solvers themselves (solve_cg, factorize,
// solve_spd) never go through them.
#pragma once

#include <cstddef>

#include "hsolve/dd.hpp"
#include "hsolve/hsolve.hpp"

namespace hsolve::kernels {

// In-place Cholesky factor of a b x b block's lower triangle; NotSpdError
// (block_row = -1, pivot) on a non-positive or NaN pivot.
void potf_block(double* d, std::size_t b);
// X L^T = X_in in place; SingularBlockError on a zero / NaN diagonal of l.
void trsm_block(double* x, const double* l, std::size_t b);
// c -= p q^T
void gemm_update(double* c, const double* p, const double* q, std::size_t b);
// lower(c) -= lower(p p^T), strict upper triangle of c untouched
void syrk_update(double* c, const double* p, std::size_t b);

// y_i = sum_j A_ij x_j for output block rows [lo, hi) (packed symmetric)
void symv_range(const BlockedSPDMatrix& a, const BlockVector& x, BlockVector& y,
                std::size_t lo, std::size_t hi);
void symv_row(const BlockedSPDMatrix& a, const BlockVector& x, BlockVector& y,
              std::size_t row);

double row_dot(const BlockVector& u, const BlockVector& v, std::size_t row);
Dd dot_rows(const BlockVector& u, const BlockVector& v, std::size_t lo, std::size_t hi);
double dot_range(const BlockVector& u, const BlockVector& v, std::size_t lo, std::size_t hi);

void axpy_range(BlockVector& y, const BlockVector& x, double alpha, std::size_t lo,
                std::size_t hi);
void xpay_range(BlockVector& s, const BlockVector& r, double beta, std::size_t lo,
                std::size_t hi);
void sub_range(BlockVector& out, const BlockVector& a, const BlockVector& b, std::size_t lo,
               std::size_t hi);

void gemv_sub(const double* m, const double* x, double* y, std::size_t b);
void gemv_transpose_sub(const double* m, const double* x, double* y, std::size_t b);
void lower_solve(const double* l, double* y, std::size_t b);
void lower_transpose_solve(const double* l, double* y, std::size_t b);

}  // namespace hsolve::kernels
