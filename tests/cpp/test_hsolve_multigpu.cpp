// Multi-GPU Runtime through the unchanged reference API: SolverConfig::gpus
// = 2 (the reference's two executors as two GPU ranks of one process),
// `fraction` as the CG row split (partition.cpp:11-22). On a one-GPU box
// both ranks share the device over the in-process transport; with two GPUs
// the same code runs over NCCL. Built and run by tests/test_cpp_shim.py.
//
// Reference assertions adapted (proj/tests/test_cg_solver.cpp:93-184,
// test_cholesky_solver.cpp:72-176): split invariance of the solution (to
// rounding: the GPU partial sums depend on the row split), the ledger
// contract of the B200 protocol, NotSpd payloads agreed by both ranks.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <string>
#include <vector>

#include "hsolve/cg_solver.hpp"
#include "hsolve/cholesky_solver.hpp"
#include "hsolve/errors.hpp"
#include "hsolve/genmat.hpp"

using namespace hsolve;

static int failures = 0;
#define CHECK(c)                                                      \
  do {                                                                \
    if (!(c)) {                                                       \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #c);        \
      ++failures;                                                     \
    }                                                                 \
  } while (0)

static SolverConfig cfg_for(std::size_t b, int gpus, double f = 0.0) {
  SolverConfig c;
  c.block_size = b;
  c.gpus = gpus;
  c.fraction = f;
  return c;
}

static double rel(const BlockVector& a, const BlockVector& b, std::size_t n) {
  double d = 0.0, nb = 0.0;
  for (std::size_t i = 0; i < n; ++i) {
    d += (a[i] - b[i]) * (a[i] - b[i]);
    nb += b[i] * b[i];
  }
  return std::sqrt(d / nb);
}

static std::size_t count_steps(const TransferLedger& l, TransferKind k, bool iterations) {
  std::size_t c = 0;
  for (const TransferEntry& e : l.entries())
    if (e.kind == k && ((e.step >= 1) == iterations)) ++c;
  return c;
}

int main() {
  const std::size_t n = 2048, b = 64;  // N = 32 block rows
  const BlockedSPDMatrix m = generate_spd(n, b, KernelParams{}, 21);
  const BlockVector rhs = generate_rhs(n, b, 21);

  // one GPU, the reference's homogeneous run
  SolverConfig c1 = cfg_for(b, 1);
  c1.record_trace = true;
  Runtime r1(c1);
  const CgResult one = solve_cg(m, rhs, c1, r1);
  CHECK(one.stats.converged);
  CHECK(r1.ledger().size() == 0);

  {  // 2 GPUs at several splits: same solution, reference residual bound
    for (double f : {0.0, 0.25, 0.5, 0.85}) {
      SolverConfig c = cfg_for(b, 2, f);
      c.record_trace = true;
      Runtime rt(c);
      const CgResult r = solve_cg(m, rhs, c, rt);
      CHECK(rt.gpus() == 2);
      CHECK(r.stats.converged);
      CHECK(r.stats.true_residual <= 2.0 * c.eps * std::sqrt(r.stats.u0));
      CHECK(std::llabs((long long)r.stats.iterations - (long long)one.stats.iterations) <= 2);
      CHECK(rel(r.x, one.x, n) <= 1e-8);
      for (std::size_t k = 0; k < 5 && k < r.stats.trace.size(); ++k) {
        CHECK(std::fabs(r.stats.trace[k].u - one.stats.trace[k].u) <=
              1e-12 * std::fabs(one.stats.trace[k].u));
        CHECK(std::fabs(r.stats.trace[k].alpha - one.stats.trace[k].alpha) <=
              1e-12 * std::fabs(one.stats.trace[k].alpha));
      }
      const std::size_t want = f > 0.0 ? partition_for_fraction(f, 32).split_row : 0;
      CHECK(r.stats.partition.split_row == want);
      CHECK(rt.ledger().size() > 0);
    }
  }
  {  // ledger contract of the row-sharded protocol, interval 5 over 12
     // iterations (test_cg_solver.cpp:148-176 counts, B200 protocol): per
     // iteration 2 subvector collectives (reduce-scatter of t carrying the
     // s.t partials, all-gather of r carrying the r.r partials), +2 on a
     // recompute; setup / exit: 2 scalar, 2 subvector, 1 result
    SolverConfig c = cfg_for(b, 2, 0.5);
    c.recompute_interval = 5;
    c.eps = 1e-300;
    c.max_iters = 12;
    Runtime rt(c);
    const CgResult r = solve_cg(m, rhs, c, rt);
    CHECK(r.stats.iterations == 12 && r.stats.recomputations == 2);
    const TransferLedger& l = rt.ledger();
    CHECK(count_steps(l, TransferKind::subvector, true) == 2 * 12 + 2 * 2);
    CHECK(count_steps(l, TransferKind::scalar, true) == 0);
    CHECK(count_steps(l, TransferKind::scalar, false) == 2);
    CHECK(count_steps(l, TransferKind::subvector, false) == 2);
    CHECK(l.count_of(TransferKind::result) == 1);
    for (const TransferEntry& e : l.entries()) CHECK(e.direction == Direction::bidirectional);
  }
  {  // Cholesky on 2 GPUs (1x2 block-cyclic) vs one GPU
    const std::size_t nc = 1024, bc = 128;
    const BlockedSPDMatrix a = generate_spd(nc, bc, KernelParams{}, 5);
    const BlockVector v = generate_rhs(nc, bc, 5);
    BlockedSPDMatrix l1(a), l2(a);
    SolverConfig s1 = cfg_for(bc, 1), s2 = cfg_for(bc, 2);
    Runtime ra(s1), rb(s2);
    factorize(l1, s1, ra);
    factorize(l2, s2, rb);
    double amax = 0.0, d = 0.0;
    for (std::size_t i = 0; i < a.value_count(); ++i) amax = std::max(amax, std::fabs(a.data()[i]));
    for (std::size_t p = 0; p < nc; ++p)
      for (std::size_t q = 0; q <= p; ++q) d = std::max(d, std::fabs(l1.element(p, q) - l2.element(p, q)));
    CHECK(d <= 1e-10 * amax);
    // the column protocol: per column j one L_jj + inverses broadcast pair
    // and N-j-1 panel broadcasts, then one status all-reduce
    const std::size_t N = nc / bc;
    std::vector<std::size_t> blocks(N, 0);
    for (const TransferEntry& e : rb.ledger().entries())
      if (e.kind == TransferKind::block && e.step >= 0) blocks[(std::size_t)e.step]++;
    for (std::size_t j = 0; j < N; ++j) CHECK(blocks[j] == 2 + (N - j - 1));
    BlockedSPDMatrix w(a);
    Runtime rc(s2);
    const SpdSolveResult sp = solve_spd(w, v, s2, rc);
    double nv = 0.0;
    for (std::size_t i = 0; i < nc; ++i) nv += v[i] * v[i];
    CHECK(sp.stats.true_residual <= 1e-10 * std::sqrt(nv));
    BlockedSPDMatrix w1(a);
    const SpdSolveResult sp1 = solve_spd(w1, v, s1, ra);
    CHECK(rel(sp.x, sp1.x, nc) <= 1e-10);
  }
  {  // NotSpd agreed by both ranks with the single-GPU payload
    BlockedSPDMatrix a = generate_spd(1024, 128, KernelParams{}, 2);
    a.set(700, 700, -5.0);
    SolverConfig c = cfg_for(128, 2);
    Runtime rt(c);
    bool thrown = false;
    try {
      factorize(a, c, rt);
    } catch (const NotSpdError& e) {
      thrown = true;
      CHECK(e.block_row() == 700 / 128 && e.pivot_index() == 700 % 128);
    }
    CHECK(thrown);
  }
  {  // shapes the distributed kernels do not serve run on rank 0's GPU
    const BlockedSPDMatrix s = generate_spd(64, 16, KernelParams{}, 3);
    const BlockVector sv = generate_rhs(64, 16, 3);
    SolverConfig c = cfg_for(16, 2, 0.5);
    Runtime rt(c);
    const CgResult r = solve_cg(s, sv, c, rt);
    CHECK(r.stats.converged);
    BlockedSPDMatrix w(s);
    const SpdSolveResult sp = solve_spd(w, sv, c, rt);
    CHECK(sp.stats.true_residual <= 1e-10 * 8.0);
  }
  std::printf(failures ? "FAILED %d\n" : "ALL PASSED\n", failures);
  return failures ? 1 : 0;
}
