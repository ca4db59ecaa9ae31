// TEST INFRASTRUCTURE ONLY (the checker, never the product).
//
// extern "C" shim over the UNMODIFIED reference `hsolve` library, compiled
// from /root/reference/proj/src by oracle/Makefile into oracle/_ref/. It lets
// the Python tests and bench.py's CPU baseline call the real reference through
// ctypes with plain pointers. Every entry point forwards to the reference API
// it names; nothing here re-implements reference arithmetic.
//
// Status convention (matches include/hs_cuda.h): 0 = ok, else
// 1 + hsolve::ErrorKind, payload in *err_a / *err_b where meaningful.
#include <cstdint>
#include <cstring>
#include <string>

#include "hsolve/block_kernels.hpp"
#include "hsolve/cg_solver.hpp"
#include "hsolve/cholesky_solver.hpp"
#include "hsolve/errors.hpp"
#include "hsolve/genmat.hpp"
#include "hsolve/matrix_io.hpp"
#include "hsolve/partition.hpp"

using namespace hsolve;

namespace {

thread_local std::string g_err;

int status_of(const Error& e) { return 1 + static_cast<int>(e.kind()); }

SolverConfig make_cfg(std::size_t b, double eps, std::size_t max_iters,
                      std::size_t recompute_interval, double fraction,
                      std::size_t workers, bool trace) {
  SolverConfig cfg;
  cfg.eps = eps;
  cfg.max_iters = max_iters;
  cfg.recompute_interval = recompute_interval;
  cfg.fraction = fraction;
  cfg.block_size = b;
  cfg.workers_a = workers;
  cfg.workers_b = workers;
  cfg.record_trace = trace;
  return cfg;
}

BlockedSPDMatrix from_packed(std::size_t n, std::size_t b, const double* v) {
  BlockedSPDMatrix m(n, b);
  std::memcpy(m.data(), v, m.value_count() * sizeof(double));
  return m;
}

BlockVector from_vec(std::size_t n, std::size_t b, const double* v) {
  BlockVector x(n, b);
  std::memcpy(x.data(), v, x.padded_n() * sizeof(double));
  return x;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// genmat.hpp:41-42
int ref_generate_spd(std::size_t n, std::size_t b, double sigma_f2,
                     double length_scale, double sigma_n2, std::size_t dim,
                     std::uint64_t seed, double* out_packed) {
  try {
    KernelParams p{sigma_f2, length_scale, sigma_n2, dim};
    BlockedSPDMatrix m = generate_spd(n, b, p, seed);
    std::memcpy(out_packed, m.data(), m.value_count() * sizeof(double));
    return 0;
  } catch (const Error& e) {
    g_err = e.what();
    return status_of(e);
  }
}

// genmat.hpp:33-38
int ref_generate_inputs(std::size_t n, std::size_t dim, std::uint64_t seed,
                        double* out) {
  try {
    auto v = generate_inputs(n, dim, seed);
    std::memcpy(out, v.data(), v.size() * sizeof(double));
    return 0;
  } catch (const Error& e) {
    g_err = e.what();
    return status_of(e);
  }
}

double ref_median_pairwise_distance(const double* pts, std::size_t n,
                                    std::size_t dim) {
  std::vector<double> v(pts, pts + n * dim);
  return median_pairwise_distance(v, n, dim);
}

// genmat.hpp:45
int ref_generate_rhs(std::size_t n, std::size_t b, std::uint64_t seed,
                     double* out) {
  BlockVector v = generate_rhs(n, b, seed);
  std::memcpy(out, v.data(), v.padded_n() * sizeof(double));
  return 0;
}

// block_kernels.hpp:34-38 (full range)
int ref_symv(std::size_t n, std::size_t b, const double* a_packed,
             const double* x, double* y) {
  BlockedSPDMatrix a = from_packed(n, b, a_packed);
  BlockVector xv = from_vec(n, b, x);
  BlockVector yv(n, b);
  kernels::symv_range(a, xv, yv, 0, a.block_rows());
  std::memcpy(y, yv.data(), yv.padded_n() * sizeof(double));
  return 0;
}

// cg_solver.hpp:48-49. stats: [iterations, recomputations, converged, u0,
// true_residual, wall_ms, compute_ms, split_row]; trace: 3 doubles/iteration.
// *ledger_counts: [scalar, subvector, initial_matrix, result] event counts.
int ref_solve_cg(std::size_t n, std::size_t b, const double* a_packed,
                 const double* rhs, double eps, std::size_t max_iters,
                 std::size_t recompute_interval, double fraction,
                 std::size_t workers, double* x_out, double* stats,
                 double* trace, std::size_t trace_cap,
                 std::uint64_t* ledger_counts) {
  try {
    BlockedSPDMatrix a = from_packed(n, b, a_packed);
    BlockVector r = from_vec(n, b, rhs);
    SolverConfig cfg = make_cfg(b, eps, max_iters, recompute_interval,
                                fraction, workers, trace != nullptr);
    Runtime rt(cfg);
    CgResult res = solve_cg(a, r, cfg, rt);
    std::memcpy(x_out, res.x.data(), res.x.padded_n() * sizeof(double));
    stats[0] = static_cast<double>(res.stats.iterations);
    stats[1] = static_cast<double>(res.stats.recomputations);
    stats[2] = res.stats.converged ? 1.0 : 0.0;
    stats[3] = res.stats.u0;
    stats[4] = res.stats.true_residual;
    stats[5] = res.stats.wall_ms;
    stats[6] = res.stats.compute_ms;
    stats[7] = static_cast<double>(res.stats.partition.split_row);
    if (trace) {
      for (std::size_t k = 0; k < res.stats.trace.size() && k < trace_cap;
           ++k) {
        trace[3 * k + 0] = res.stats.trace[k].u;
        trace[3 * k + 1] = res.stats.trace[k].alpha;
        trace[3 * k + 2] = res.stats.trace[k].beta;
      }
    }
    if (ledger_counts) {
      const auto& l = rt.ledger();
      ledger_counts[0] = l.count_of(TransferKind::scalar);
      ledger_counts[1] = l.count_of(TransferKind::subvector);
      ledger_counts[2] = l.count_of(TransferKind::initial_matrix);
      ledger_counts[3] = l.count_of(TransferKind::result);
    }
    return 0;
  } catch (const Error& e) {
    g_err = e.what();
    return status_of(e);
  }
}

// cholesky_solver.hpp:44-45. In place on a_packed. On not_spd, err_a =
// block row, err_b = pivot. stats: [factor_ms, compute_ms].
int ref_factorize(std::size_t n, std::size_t b, double* a_packed,
                  double fraction, std::size_t workers, double* stats,
                  long long* err_a, long long* err_b) {
  try {
    BlockedSPDMatrix a = from_packed(n, b, a_packed);
    SolverConfig cfg = make_cfg(b, 1e-6, 500, 50, fraction, workers, false);
    Runtime rt(cfg);
    FactorizeStats st = factorize(a, cfg, rt);
    std::memcpy(a_packed, a.data(), a.value_count() * sizeof(double));
    if (stats) {
      stats[0] = st.factor_ms;
      stats[1] = st.compute_ms;
    }
    return 0;
  } catch (const NotSpdError& e) {
    g_err = e.what();
    if (err_a) *err_a = e.block_row();
    if (err_b) *err_b = static_cast<long long>(e.pivot_index());
    return status_of(e);
  } catch (const Error& e) {
    g_err = e.what();
    return status_of(e);
  }
}

// cholesky_solver.hpp:57-58. a_packed is destroyed (holds L). stats:
// [factor_ms, solve_ms, wall_ms, compute_ms, true_residual].
int ref_solve_spd(std::size_t n, std::size_t b, double* a_packed,
                  const double* rhs, double fraction, std::size_t workers,
                  double* x_out, double* stats) {
  try {
    BlockedSPDMatrix a = from_packed(n, b, a_packed);
    BlockVector r = from_vec(n, b, rhs);
    SolverConfig cfg = make_cfg(b, 1e-6, 500, 50, fraction, workers, false);
    Runtime rt(cfg);
    SpdSolveResult res = solve_spd(a, r, cfg, rt);
    std::memcpy(a_packed, a.data(), a.value_count() * sizeof(double));
    std::memcpy(x_out, res.x.data(), res.x.padded_n() * sizeof(double));
    stats[0] = res.stats.factor_ms;
    stats[1] = res.stats.solve_ms;
    stats[2] = res.stats.wall_ms;
    stats[3] = res.stats.compute_ms;
    stats[4] = res.stats.true_residual;
    return 0;
  } catch (const Error& e) {
    g_err = e.what();
    return status_of(e);
  }
}

// cholesky_solver.hpp:50-52
int ref_forward_substitute(std::size_t n, std::size_t b, const double* l,
                           const double* rhs, double* y_out) {
  try {
    BlockedSPDMatrix lm = from_packed(n, b, l);
    BlockVector y = forward_substitute(lm, from_vec(n, b, rhs));
    std::memcpy(y_out, y.data(), y.padded_n() * sizeof(double));
    return 0;
  } catch (const Error& e) {
    g_err = e.what();
    return status_of(e);
  }
}

int ref_back_substitute(std::size_t n, std::size_t b, const double* l,
                        const double* y, double* x_out) {
  try {
    BlockedSPDMatrix lm = from_packed(n, b, l);
    BlockVector x = back_substitute(lm, from_vec(n, b, y));
    std::memcpy(x_out, x.data(), x.padded_n() * sizeof(double));
    return 0;
  } catch (const Error& e) {
    g_err = e.what();
    return status_of(e);
  }
}

// block_kernels.hpp:17-31 single-block kernels.
int ref_potf_block(double* d, std::size_t b, long long* pivot) {
  try {
    kernels::potf_block(d, b);
    return 0;
  } catch (const NotSpdError& e) {
    if (pivot) *pivot = static_cast<long long>(e.pivot_index());
    return status_of(e);
  }
}
int ref_trsm_block(double* x, const double* l, std::size_t b) {
  try {
    kernels::trsm_block(x, l, b);
    return 0;
  } catch (const Error& e) {
    return status_of(e);
  }
}
void ref_gemm_update(double* c, const double* p, const double* q,
                     std::size_t b) {
  kernels::gemm_update(c, p, q, b);
}
void ref_syrk_update(double* c, const double* p, std::size_t b) {
  kernels::syrk_update(c, p, b);
}

// partition.hpp:22-27
std::size_t ref_partition_for_fraction(double f, std::size_t rows) {
  return partition_for_fraction(f, rows).split_row;
}
std::size_t ref_cholesky_border(double f, std::size_t col, std::size_t rows) {
  return cholesky_border(f, col, rows);
}

// matrix_io.hpp:16-19 (BSPD1 files). load: *n, *b set on success; the
// packed values are copied to `out` when it is non-null and `cap` matches.
int ref_save_matrix(std::size_t n, std::size_t b, const double* v, const char* path) {
  try {
    save_matrix(from_packed(n, b, v), path);
    return 0;
  } catch (const Error& e) {
    g_err = e.what();
    return status_of(e);
  }
}
int ref_load_matrix(const char* path, std::size_t* n, std::size_t* b, double* out,
                    std::size_t cap, std::int64_t* err_a, std::int64_t* err_b) {
  try {
    const BlockedSPDMatrix m = load_matrix(path);
    *n = m.n();
    *b = m.block_size();
    if (out && cap == m.value_count())
      std::memcpy(out, m.data(), cap * sizeof(double));
    return 0;
  } catch (const TruncatedFileError& e) {
    g_err = e.what();
    *err_a = (std::int64_t)e.expected_bytes();
    *err_b = (std::int64_t)e.actual_bytes();
    return status_of(e);
  } catch (const Error& e) {
    g_err = e.what();
    return status_of(e);
  }
}
int ref_save_vector(std::size_t n, std::size_t b, const double* v, const char* path) {
  try {
    save_vector(from_vec(n, b, v), path);
    return 0;
  } catch (const Error& e) {
    g_err = e.what();
    return status_of(e);
  }
}

}  // extern "C"
