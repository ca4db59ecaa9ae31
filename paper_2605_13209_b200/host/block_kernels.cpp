// hsolve::kernels (include/hsolve/block_kernels.hpp): the reference's
// per-block kernel API (block_kernels.hpp:16-74) on host buffers, each call
// one round trip to the default context's GPU: copy the operands in, run the
// sm_100a kernel (hs_block_exact, hs_trsm_tiles, hs_symv_exact,
// hs_block_vec_op, hs_range_op), copy the result out. No arithmetic runs on
// the host except the reference's own double-double combine of per-row dots
// (dot_rows, dd.hpp).
#include "hsolve/block_kernels.hpp"

#include <cstring>
#include <vector>

#include "hs_cuda.h"
#include "host_internal.hpp"

namespace hsolve::kernels {

namespace {

using detail::check;
using detail::default_ctx;

// device scratch for one call, freed on every exit path
struct DevBuf {
  hs_ctx* ctx;
  void* p = nullptr;
  DevBuf(hs_ctx* c, std::size_t bytes) : ctx(c) { check(hs_device_alloc(c, bytes, &p)); }
  ~DevBuf() { hs_device_free(ctx, p); }
  double* d() const { return static_cast<double*>(p); }
};

void to_dev(hs_ctx* c, double* dst, const double* src, std::size_t n) {
  check(hs_memcpy(c, dst, src, n * sizeof(double)));
}
void to_host(hs_ctx* c, double* dst, const double* src, std::size_t n) {
  check(hs_memcpy(c, dst, src, n * sizeof(double)));
}

void same_shape(const BlockVector& a, const BlockVector& b) {
  if (a.n() != b.n() || a.block_size() != b.block_size())
    throw ConfigError("vector shapes do not match");
}

void check_rows(const BlockVector& v, std::size_t lo, std::size_t hi) {
  if (lo > hi || hi > v.block_rows()) throw std::out_of_range("block-row range out of range");
}

// one range op over block rows [lo, hi) of padded vectors
void range(int op, BlockVector& out, const BlockVector* u, const BlockVector* v, double alpha,
           std::size_t lo, std::size_t hi) {
  hs_ctx* c = default_ctx();
  const std::size_t pn = out.padded_n();
  DevBuf dout(c, pn * sizeof(double)), du(c, pn * sizeof(double)),
      dv(c, (v ? pn : 1) * sizeof(double));
  if (op != 0) to_dev(c, dout.d(), out.data(), pn);
  if (u) to_dev(c, du.d(), u->data(), pn);
  if (v) to_dev(c, dv.d(), v->data(), pn);
  check(hs_range_op(c, op, dout.d(), du.d(), dv.d(), alpha, lo, hi, out.block_size()));
  to_host(c, out.data(), dout.d(), pn);
}

std::vector<double> row_dots(const BlockVector& u, const BlockVector& v, std::size_t lo,
                             std::size_t hi) {
  same_shape(u, v);
  check_rows(u, lo, hi);
  BlockVector out(u.n(), u.block_size());  // row i's dot at index i
  range(0, out, &u, &v, 0.0, lo, hi);
  return std::vector<double>(out.data() + lo, out.data() + hi);
}

}  // namespace

void potf_block(double* d, std::size_t b) {
  hs_ctx* c = default_ctx();
  DevBuf dd(c, b * b * sizeof(double));
  to_dev(c, dd.d(), d, b * b);
  int64_t bad = -1;
  const hs_status s = hs_block_exact(c, 0, dd.d(), nullptr, nullptr, b, &bad);
  if (s == HS_ERR_NOT_SPD) throw NotSpdError(-1, (std::size_t)bad);
  check(s);
  to_host(c, d, dd.d(), b * b);  // the kernel leaves the strict upper triangle as it was
}

void trsm_block(double* x, const double* l, std::size_t b) {
  hs_ctx* c = default_ctx();
  DevBuf dx(c, b * b * sizeof(double)), dl(c, b * b * sizeof(double));
  to_dev(c, dx.d(), x, b * b);
  to_dev(c, dl.d(), l, b * b);
  const hs_status s = hs_trsm_tiles(c, dx.d(), dl.d(), b, 1);
  if (s == HS_ERR_SINGULAR_BLOCK) {
    int64_t pa = -1, pb = -1;
    hs_last_error_payload(&pa, &pb);
    throw SingularBlockError((std::size_t)pb);
  }
  check(s);
  to_host(c, x, dx.d(), b * b);
}

void gemm_update(double* cc, const double* p, const double* q, std::size_t b) {
  hs_ctx* c = default_ctx();
  DevBuf dc(c, b * b * sizeof(double)), dp(c, b * b * sizeof(double)),
      dq(c, b * b * sizeof(double));
  to_dev(c, dc.d(), cc, b * b);
  to_dev(c, dp.d(), p, b * b);
  to_dev(c, dq.d(), q, b * b);
  check(hs_block_exact(c, 1, dc.d(), dp.d(), dq.d(), b, nullptr));
  to_host(c, cc, dc.d(), b * b);
}

void syrk_update(double* cc, const double* p, std::size_t b) {
  hs_ctx* c = default_ctx();
  DevBuf dc(c, b * b * sizeof(double)), dp(c, b * b * sizeof(double));
  to_dev(c, dc.d(), cc, b * b);
  to_dev(c, dp.d(), p, b * b);
  check(hs_block_exact(c, 2, dc.d(), dp.d(), dp.d(), b, nullptr));
  to_host(c, cc, dc.d(), b * b);
}

void symv_range(const BlockedSPDMatrix& a, const BlockVector& x, BlockVector& y,
                std::size_t lo, std::size_t hi) {
  if (x.n() != a.n() || x.block_size() != a.block_size())
    throw ConfigError("matrix and vector shapes do not match");
  same_shape(x, y);
  check_rows(y, lo, hi);
  if (hi == lo) return;
  hs_ctx* c = default_ctx();
  const std::size_t pn = x.padded_n(), b = a.block_size();
  DevBuf da(c, a.value_count() * sizeof(double)), dx(c, pn * sizeof(double)),
      dy(c, pn * sizeof(double));
  to_dev(c, da.d(), a.data(), a.value_count());
  to_dev(c, dx.d(), x.data(), pn);
  check(hs_symv_exact(c, da.d(), dx.d(), dy.d(), a.n(), b, lo, hi));
  to_host(c, y.data() + lo * b, dy.d() + lo * b, (hi - lo) * b);
}

void symv_row(const BlockedSPDMatrix& a, const BlockVector& x, BlockVector& y,
              std::size_t row) {
  symv_range(a, x, y, row, row + 1);
}

double row_dot(const BlockVector& u, const BlockVector& v, std::size_t row) {
  return row_dots(u, v, row, row + 1)[0];
}

Dd dot_rows(const BlockVector& u, const BlockVector& v, std::size_t lo, std::size_t hi) {
  Dd acc;
  for (double p : row_dots(u, v, lo, hi)) acc = dd_add(acc, p);  // block_kernels.cpp:108-112
  return acc;
}

double dot_range(const BlockVector& u, const BlockVector& v, std::size_t lo, std::size_t hi) {
  return dd_value(dot_rows(u, v, lo, hi));
}

void axpy_range(BlockVector& y, const BlockVector& x, double alpha, std::size_t lo,
                std::size_t hi) {
  same_shape(y, x);
  check_rows(y, lo, hi);
  range(1, y, &x, nullptr, alpha, lo, hi);
}

void xpay_range(BlockVector& s, const BlockVector& r, double beta, std::size_t lo,
                std::size_t hi) {
  same_shape(s, r);
  check_rows(s, lo, hi);
  range(2, s, &r, nullptr, beta, lo, hi);
}

void sub_range(BlockVector& out, const BlockVector& a, const BlockVector& b, std::size_t lo,
               std::size_t hi) {
  same_shape(out, a);
  same_shape(out, b);
  check_rows(out, lo, hi);
  range(3, out, &a, &b, 0.0, lo, hi);
}

namespace {
void block_vec(int op, const double* m, const double* x, double* y, std::size_t b) {
  hs_ctx* c = default_ctx();
  DevBuf dm(c, b * b * sizeof(double)), dx(c, b * sizeof(double)), dy(c, b * sizeof(double));
  to_dev(c, dm.d(), m, b * b);
  if (x) to_dev(c, dx.d(), x, b);
  to_dev(c, dy.d(), y, b);
  const hs_status s = hs_block_vec_op(c, op, dm.d(), x ? dx.d() : nullptr, dy.d(), b);
  if (s == HS_ERR_SINGULAR_BLOCK) {
    int64_t pa = -1, pb = -1;
    hs_last_error_payload(&pa, &pb);
    throw SingularBlockError((std::size_t)pb);
  }
  check(s);
  to_host(c, y, dy.d(), b);
}
}  // namespace

void gemv_sub(const double* m, const double* x, double* y, std::size_t b) {
  block_vec(0, m, x, y, b);
}
void gemv_transpose_sub(const double* m, const double* x, double* y, std::size_t b) {
  block_vec(1, m, x, y, b);
}
void lower_solve(const double* l, double* y, std::size_t b) { block_vec(2, l, nullptr, y, b); }
void lower_transpose_solve(const double* l, double* y, std::size_t b) {
  block_vec(3, l, nullptr, y, b);
}

}  // namespace hsolve::kernels
