// The kernel-level drop-in (include/hsolve/block_kernels.hpp, dd.hpp) against
// the reference's own known answers (proj/tests/test_block_kernels.cpp:33-370)
// and bitwise against in-test triple loops in the reference's order. Built
// and run on a GPU box by tests/test_cpp_shim.py.
#include <cmath>
#include <cstdio>
#include <random>
#include <vector>

#include "hsolve/block_kernels.hpp"
#include "hsolve/dd.hpp"
#include "hsolve/errors.hpp"
#include "hsolve/genmat.hpp"

using namespace hsolve;
namespace k = hsolve::kernels;

static int failures = 0;
#define CHECK(c)                                                      \
  do {                                                                \
    if (!(c)) {                                                       \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #c);        \
      ++failures;                                                     \
    }                                                                 \
  } while (0)

static std::vector<double> randv(std::size_t n, unsigned seed) {
  std::mt19937_64 g(seed);
  std::uniform_real_distribution<double> u(-1.0, 1.0);
  std::vector<double> v(n);
  for (double& x : v) x = u(g);
  return v;
}

static bool close(double a, double b, double tol) { return std::fabs(a - b) <= tol; }

int main() {
  const double s2 = std::sqrt(2.0);
  {  // potf_block closed forms (test_block_kernels.cpp:33-55)
    std::vector<double> d = {4.0, 2.0, 2.0, 3.0};
    k::potf_block(d.data(), 2);
    CHECK(d[0] == 2.0 && d[2] == 1.0 && close(d[3], s2, 1e-15) && d[1] == 2.0);
    std::vector<double> bad = {1.0, 2.0, 2.0, 1.0};
    bool thrown = false;
    try {
      k::potf_block(bad.data(), 2);
    } catch (const NotSpdError& e) {
      thrown = true;
      CHECK(e.pivot_index() == 1 && e.block_row() == -1);
    }
    CHECK(thrown);
  }
  {  // potf_block bitwise vs the row-wise loops, b = 37 (random SPD: M M^T + b I)
    const std::size_t b = 37;
    std::vector<double> m = randv(b * b, 5), a(b * b, 0.0);
    for (std::size_t r = 0; r < b; ++r)
      for (std::size_t c = 0; c < b; ++c) {
        double acc = 0.0;
        for (std::size_t t = 0; t < b; ++t) acc += m[r * b + t] * m[c * b + t];
        a[r * b + c] = acc + (r == c ? (double)b : 0.0);
      }
    std::vector<double> ref = a, got = a;
    for (std::size_t p = 0; p < b; ++p) {
      for (std::size_t q = 0; q < p; ++q) {
        double acc = ref[p * b + q];
        for (std::size_t t = 0; t < q; ++t) acc -= ref[p * b + t] * ref[q * b + t];
        ref[p * b + q] = acc / ref[q * b + q];
      }
      double acc = ref[p * b + p];
      for (std::size_t t = 0; t < p; ++t) acc -= ref[p * b + t] * ref[p * b + t];
      ref[p * b + p] = std::sqrt(acc);
    }
    k::potf_block(got.data(), b);
    CHECK(got == ref);
  }
  {  // trsm_block closed form (test_block_kernels.cpp:86-102) + bitwise
    std::vector<double> x = {2.0, 0.0, 0.0, 2.0}, l = {2.0, 0.0, 1.0, s2};
    k::trsm_block(x.data(), l.data(), 2);
    CHECK(close(x[0], 1.0, 1e-15) && close(x[1], -s2 / 2, 1e-15) && close(x[2], 0.0, 1e-15) &&
          close(x[3], s2, 1e-15));
    const std::size_t b = 19;
    std::vector<double> L = randv(b * b, 7), X = randv(b * b, 8);
    for (std::size_t r = 0; r < b; ++r) L[r * b + r] = 2.0 + r;
    std::vector<double> ref = X;
    for (std::size_t r = 0; r < b; ++r)
      for (std::size_t c = 0; c < b; ++c) {
        double acc = ref[r * b + c];
        for (std::size_t t = 0; t < c; ++t) acc -= ref[r * b + t] * L[c * b + t];
        ref[r * b + c] = acc / L[c * b + c];
      }
    k::trsm_block(X.data(), L.data(), b);
    CHECK(X == ref);
    std::vector<double> sing = {1.0, 0.0, 1.0, 0.0}, y = {1.0, 1.0, 1.0, 1.0};
    bool thrown = false;
    try {
      k::trsm_block(y.data(), sing.data(), 2);
    } catch (const SingularBlockError& e) {
      thrown = e.diagonal_index() == 1;
    }
    CHECK(thrown);
  }
  {  // gemm / syrk worked examples (test_block_kernels.cpp:150-183) + bitwise
    std::vector<double> c = {1.0, 0.0, 0.0, 1.0}, p = {1.0, 2.0, 3.0, 4.0}, q = {1.0, 0.0, 0.0, 1.0};
    k::gemm_update(c.data(), p.data(), q.data(), 2);
    CHECK((c == std::vector<double>{0.0, -2.0, -3.0, -3.0}));
    std::vector<double> s = {5.0, 42.0, 2.0, 5.0}, o = {1.0, 1.0, 1.0, 1.0};
    k::syrk_update(s.data(), o.data(), 2);
    CHECK((s == std::vector<double>{3.0, 42.0, 0.0, 3.0}));
    const std::size_t b = 16;
    std::vector<double> C = randv(b * b, 2), P = randv(b * b, 3), Q = randv(b * b, 4), R = C;
    for (std::size_t r = 0; r < b; ++r)
      for (std::size_t col = 0; col < b; ++col) {
        double acc = 0.0;
        for (std::size_t t = 0; t < b; ++t) acc += P[r * b + t] * Q[col * b + t];
        R[r * b + col] -= acc;
      }
    k::gemm_update(C.data(), P.data(), Q.data(), b);
    CHECK(C == R);
  }
  {  // symv: 1x1 worked example and bitwise vs symv_row's loops (45, 8)
    BlockedSPDMatrix m(2, 1);
    m.set(0, 0, 2.0);
    m.set(1, 0, 1.0);
    m.set(1, 1, 3.0);
    BlockVector x(2, 1), y(2, 1);
    x[0] = x[1] = 1.0;
    k::symv_range(m, x, y, 0, 2);
    CHECK(y[0] == 3.0 && y[1] == 4.0);
    const BlockedSPDMatrix a = generate_spd(45, 8, KernelParams{}, 17);
    BlockVector v(45, 8), out(45, 8), whole(45, 8);
    const std::vector<double> xv = randv(45, 10);
    for (std::size_t i = 0; i < 45; ++i) v[i] = xv[i];
    k::symv_range(a, v, whole, 0, a.block_rows());
    const std::size_t N = a.block_rows(), b = 8;
    bool same = true;
    for (std::size_t i = 0; i < N; ++i)
      for (std::size_t r = 0; r < b; ++r) {
        double acc = 0.0;
        for (std::size_t j = 0; j < N; ++j)
          for (std::size_t c = 0; c < b; ++c) {
            double val;
            if (j < i) val = a.block(i, j)[r * b + c];
            else if (j == i) val = c <= r ? a.block(i, i)[r * b + c] : a.block(i, i)[c * b + r];
            else val = a.block(j, i)[c * b + r];
            acc += val * v[j * b + c];
          }
        same &= whole[i * b + r] == acc;
      }
    CHECK(same);
    y[0] = 42.0;
    k::symv_range(m, x, y, 0, 0);  // empty range: no writes
    CHECK(y[0] == 42.0);
    k::symv_range(a, v, out, 0, 2);
    k::symv_range(a, v, out, 2, N);
    bool cat = true;
    for (std::size_t i = 0; i < out.padded_n(); ++i) cat &= out.data()[i] == whole.data()[i];
    CHECK(cat);
  }
  {  // dots (test_block_kernels.cpp:288-310) and range updates
    BlockVector u(3, 1), v(3, 1);
    u[0] = 1.0; u[1] = 2.0; u[2] = 3.0;
    v[0] = 4.0; v[1] = 5.0; v[2] = 6.0;
    CHECK(k::dot_range(u, v, 0, 3) == 32.0);
    CHECK(k::row_dot(u, v, 2) == 18.0);
    BlockVector p(96, 8), q(96, 8);
    const std::vector<double> pv = randv(96, 12), qv = randv(96, 13);
    for (std::size_t i = 0; i < 96; ++i) {
      p[i] = pv[i];
      q[i] = qv[i];
    }
    const Dd whole = k::dot_rows(p, q, 0, 12);
    for (std::size_t r = 0; r <= 12; r += 3)
      CHECK(dd_value(dd_add(k::dot_rows(p, q, 0, r), k::dot_rows(p, q, r, 12))) ==
            dd_value(whole));
    BlockVector y = p;
    k::axpy_range(y, q, 0.5, 1, 11);
    bool ok = true;
    for (std::size_t i = 0; i < 96; ++i)
      ok &= y[i] == ((i >= 8 && i < 88) ? p[i] + 0.5 * q[i] : p[i]);
    CHECK(ok);
    BlockVector s = p;
    k::xpay_range(s, q, 2.0, 0, 12);
    ok = true;
    for (std::size_t i = 0; i < 96; ++i) ok &= s[i] == q[i] + 2.0 * p[i];
    CHECK(ok);
    BlockVector d(96, 8);
    k::sub_range(d, p, q, 0, 12);
    ok = true;
    for (std::size_t i = 0; i < 96; ++i) ok &= d[i] == p[i] - q[i];
    CHECK(ok);
  }
  {  // triangular block solves + gemv (test_block_kernels.cpp:340-370)
    std::vector<double> l = {2.0, 0.0, 1.0, s2}, y = {2.0, 1.0 + s2};
    k::lower_solve(l.data(), y.data(), 2);
    CHECK(close(y[0], 1.0, 1e-15) && close(y[1], 1.0, 1e-15));
    k::lower_transpose_solve(l.data(), y.data(), 2);
    CHECK(close(4.0 * y[0] + 2.0 * y[1], 2.0, 1e-12) && close(2.0 * y[0] + 3.0 * y[1], 1.0 + s2, 1e-12));
    std::vector<double> bad = {1.0, 0.0, 1.0, 0.0}, z = {1.0, 1.0};
    bool t1 = false, t2 = false;
    try {
      k::lower_solve(bad.data(), z.data(), 2);
    } catch (const SingularBlockError&) {
      t1 = true;
    }
    try {
      k::lower_transpose_solve(bad.data(), z.data(), 2);
    } catch (const SingularBlockError&) {
      t2 = true;
    }
    CHECK(t1 && t2);
    const std::size_t b = 13;
    std::vector<double> M = randv(b * b, 21), xx = randv(b, 22), g1 = randv(b, 23), g2 = g1;
    std::vector<double> r1 = g1, r2 = g1;
    for (std::size_t r = 0; r < b; ++r) {
      double a1 = 0.0, a2 = 0.0;
      for (std::size_t c = 0; c < b; ++c) {
        a1 += M[r * b + c] * xx[c];
        a2 += M[c * b + r] * xx[c];
      }
      r1[r] -= a1;
      r2[r] -= a2;
    }
    k::gemv_sub(M.data(), xx.data(), g1.data(), b);
    k::gemv_transpose_sub(M.data(), xx.data(), g2.data(), b);
    CHECK(g1 == r1 && g2 == r2);
  }
  std::printf(failures ? "FAILED %d\n" : "ALL PASSED\n", failures);
  return failures ? 1 : 0;
}
