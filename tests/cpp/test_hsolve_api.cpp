// Drop-in check of the C++ shim (libhsolve_b200.so): reference-style
// assertions (after proj/tests/test_cg_solver.cpp, test_cholesky_solver.cpp,
// test_genmat.cpp) written against the unchanged reference API names.
// Built and run by tests/test_cpp_shim.py on a GPU box.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <string>

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

static SolverConfig cfg_for(std::size_t b) {
  SolverConfig c;
  c.block_size = b;
  return c;
}

int main() {
  {  // identity converges in one iteration (test_cg_solver.cpp:28-39)
    const BlockedSPDMatrix id = BlockedSPDMatrix::identity(64, 16);
    const BlockVector rhs = generate_rhs(64, 16, 1);
    SolverConfig cfg = cfg_for(16);
    Runtime rt(cfg);
    const CgResult r = solve_cg(id, rhs, cfg, rt);
    CHECK(r.stats.iterations == 1 && r.stats.converged);
    for (std::size_t i = 0; i < 64; ++i) CHECK(r.x[i] == rhs[i]);
    CHECK(rt.ledger().size() == 0);
  }
  {  // generated system: residual bound (test_cg_solver.cpp:76-91)
    const BlockedSPDMatrix m = generate_spd(1024, 128, KernelParams{}, 42);
    const BlockVector rhs = generate_rhs(1024, 128, 42);
    SolverConfig cfg = cfg_for(128);
    Runtime rt(cfg);
    const CgResult r = solve_cg(m, rhs, cfg, rt);
    CHECK(r.stats.converged);
    CHECK(r.stats.iterations >= 28 && r.stats.iterations <= 32);  // reference: 30
    CHECK(r.stats.true_residual <= 2.0 * cfg.eps * std::sqrt(r.stats.u0));
    BlockedSPDMatrix work(m);
    const SpdSolveResult s = solve_spd(work, rhs, cfg, rt);
    double nr = 0.0;
    for (std::size_t i = 0; i < 1024; ++i) nr += rhs[i] * rhs[i];
    CHECK(s.stats.true_residual <= 1e-10 * std::sqrt(nr));
    double dx = 0.0, nx = 0.0;
    for (std::size_t i = 0; i < 1024; ++i) {
      dx += (s.x[i] - r.x[i]) * (s.x[i] - r.x[i]);
      nx += s.x[i] * s.x[i];
    }
    CHECK(std::sqrt(dx) <= 1e-5 * std::sqrt(nx));  // CG vs Cholesky
  }
  {  // closed-form 2x2 factor (test_cholesky_solver.cpp:35-50)
    BlockedSPDMatrix m(2, 1);
    m.set(0, 0, 4.0);
    m.set(1, 0, 2.0);
    m.set(1, 1, 3.0);
    SolverConfig cfg = cfg_for(1);
    Runtime rt(cfg);
    factorize(m, cfg, rt);
    CHECK(m.block(0, 0)[0] == 2.0 && m.block(1, 0)[0] == 1.0);
    CHECK(std::fabs(m.block(1, 1)[0] - std::sqrt(2.0)) <= 1e-15);
  }
  {  // not SPD reports the failing column (test_cholesky_solver.cpp:208-224)
    BlockedSPDMatrix m = generate_spd(64, 16, KernelParams{}, 2);
    m.set(40, 40, -5.0);
    SolverConfig cfg = cfg_for(16);
    Runtime rt(cfg);
    bool thrown = false;
    try {
      factorize(m, cfg, rt);
    } catch (const NotSpdError& e) {
      thrown = true;
      CHECK(e.block_row() == 2 && e.pivot_index() == 8);
      CHECK(std::string(to_string(e.kind())) == "not_spd");
    }
    CHECK(thrown);
  }
  {  // substitutions + singular diagonal (test_cholesky_solver.cpp:226-282)
    BlockedSPDMatrix l = BlockedSPDMatrix::identity(4, 2);
    l.set(2, 2, 0.0);
    BlockVector rhs(4, 2);
    rhs[0] = 1.0;
    bool thrown = false;
    try {
      forward_substitute(l, rhs);
    } catch (const SingularBlockError&) {
      thrown = true;
    }
    CHECK(thrown);
  }
  {  // config errors (solver_config.cpp:9-26)
    SolverConfig bad;
    bad.eps = 0.0;
    bool thrown = false;
    try {
      bad.validate();
    } catch (const ConfigError&) {
      thrown = true;
    }
    CHECK(thrown);
    CHECK(partition_for_fraction(0.5, 7).split_row == 4);
    CHECK(CholeskyPlan::for_fraction(0.5, 8).borders.size() == 8);
  }
  std::printf(failures ? "FAILED %d\n" : "ALL PASSED\n", failures);
  return failures ? 1 : 0;
}
