// libhsolve_b200.so: the reference hsolve C++ API (include/hsolve/hsolve.hpp)
// implemented on the B200 C ABI (include/hs_cuda.h). Host-side bookkeeping
// only; every arithmetic step on a matrix runs in libhsolve_cuda.so.
#include "hsolve/hsolve.hpp"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <map>
#include <mutex>
#include <tuple>

#include "hs_cuda.h"
#include "host_internal.hpp"

namespace hsolve {

namespace detail {

[[noreturn]] void raise(hs_status s) {
  const std::string msg = hs_last_error();
  int64_t a = -1, b = -1;
  hs_last_error_payload(&a, &b);
  switch (s) {
    case HS_ERR_CONFIG: throw ConfigError(msg);
    case HS_ERR_NOT_SPD: throw NotSpdError(a, (std::size_t)b);
    case HS_ERR_SINGULAR_BLOCK: throw SingularBlockError((std::size_t)b);
    case HS_ERR_NUMERICAL: throw NumericalError(msg);
    case HS_ERR_RESIDENCY: throw ResidencyError(msg);
    case HS_ERR_FORMAT: throw FormatError(msg);
    case HS_ERR_VERSION_MISMATCH: throw VersionMismatchError((unsigned)a, (unsigned)b);
    case HS_ERR_TRUNCATED_FILE: throw TruncatedFileError((std::uint64_t)a, (std::uint64_t)b);
    case HS_ERR_IO: throw IoError(msg);
    default: throw DeviceError(msg);
  }
}

void check(hs_status s) {
  if (s != HS_OK) raise(s);
}

}  // namespace detail

// Context for the reference entry points that take no Runtime
// (forward_substitute / back_substitute, generate_spd, hsolve::kernels).
hs_ctx* detail::default_ctx() {
  static std::once_flag once;
  static hs_ctx* ctx = nullptr;
  static hs_status st = HS_OK;
  std::call_once(once, [] { st = hs_ctx_create(0, nullptr, &ctx); });
  check(st);
  return ctx;
}

namespace {

using detail::check;
using detail::default_ctx;

// The plan a factorization reports: the GPU paths never run the reference's
// moving-border CPU/GPU split (one GPU, or a static 2D block-cyclic grid),
// so no borders and no shift events -- only the requested fraction.
CholeskyPlan plan_for(const SolverConfig& cfg, std::size_t) {
  CholeskyPlan p;
  p.fraction = cfg.fraction;
  return p;
}

}  // namespace

// ---- errors ----------------------------------------------------------------

const char* to_string(ErrorKind k) {
  switch (k) {
    case ErrorKind::config: return "config_error";
    case ErrorKind::not_spd: return "not_spd";
    case ErrorKind::singular_block: return "singular_block";
    case ErrorKind::numerical: return "numerical_error";
    case ErrorKind::not_converged: return "not_converged";
    case ErrorKind::residency: return "residency_error";
    case ErrorKind::format: return "format_error";
    case ErrorKind::version_mismatch: return "version_mismatch";
    case ErrorKind::truncated_file: return "truncated_file";
    case ErrorKind::io: return "io_error";
  }
  return "unknown";
}

NotSpdError::NotSpdError(std::ptrdiff_t block_row, std::size_t pivot)
    : Error(ErrorKind::not_spd,
            "matrix is not positive definite (block row " +
                std::to_string(block_row) + ", pivot " + std::to_string(pivot) +
                ")"),
      row_(block_row),
      pivot_(pivot) {}

SingularBlockError::SingularBlockError(std::size_t index)
    : Error(ErrorKind::singular_block,
            "triangular block has zero or NaN diagonal at index " +
                std::to_string(index)),
      index_(index) {}

// ---- storage ---------------------------------------------------------------

std::size_t block_index(std::size_t i, std::size_t j, std::size_t rows) {
  if (i >= rows || j > i)
    throw std::out_of_range("block_index(" + std::to_string(i) + ", " +
                            std::to_string(j) + ") out of range for " +
                            std::to_string(rows) + " block rows");
  return i * (i + 1) / 2 + j;
}

BlockedSPDMatrix::BlockedSPDMatrix(std::size_t n, std::size_t b)
    : n_(n), b_(b), rows_(b ? (n + b - 1) / b : 0) {
  if (n == 0 || b == 0)
    throw ConfigError("matrix size and block size must be positive");
  v_.assign(block_count() * b * b, 0.0);
  apply_identity_padding();
}

BlockedSPDMatrix BlockedSPDMatrix::identity(std::size_t n, std::size_t b) {
  BlockedSPDMatrix m(n, b);
  for (std::size_t i = 0; i < m.rows_; ++i) {
    double* d = m.block(i, i);
    for (std::size_t r = 0; r < b; ++r) d[r * b + r] = 1.0;
  }
  return m;
}

double BlockedSPDMatrix::element(std::size_t p, std::size_t q) const {
  if (p >= n_ || q >= n_) throw std::out_of_range("element out of range");
  if (p < q) std::swap(p, q);
  return block(p / b_, q / b_)[(p % b_) * b_ + q % b_];
}

void BlockedSPDMatrix::set(std::size_t p, std::size_t q, double value) {
  if (p >= n_ || q >= n_) throw std::out_of_range("set out of range");
  if (p < q) std::swap(p, q);
  block(p / b_, q / b_)[(p % b_) * b_ + q % b_] = value;
}

void BlockedSPDMatrix::apply_identity_padding() {
  if (pad() == 0) return;
  const std::size_t last = rows_ - 1;
  for (std::size_t j = 0; j <= last; ++j) {
    double* d = block(last, j);
    for (std::size_t r = 0; r < b_; ++r) {
      const std::size_t p = last * b_ + r;
      if (p < n_) continue;
      for (std::size_t c = 0; c < b_; ++c) d[r * b_ + c] = (p == j * b_ + c);
    }
  }
}

BlockVector::BlockVector(std::size_t n, std::size_t b)
    : n_(n), b_(b), rows_(b ? (n + b - 1) / b : 0) {
  if (n == 0 || b == 0)
    throw ConfigError("vector size and block size must be positive");
  v_.assign(rows_ * b_, 0.0);
}

// ---- config / partition / ledger -------------------------------------------

void SolverConfig::validate() const {
  if (!(eps > 0.0)) throw ConfigError("eps must be positive, got " + std::to_string(eps));
  if (!(fraction >= 0.0 && fraction <= 1.0))
    throw ConfigError("fraction must be in [0, 1], got " + std::to_string(fraction));
  if (block_size == 0) throw ConfigError("block size must be positive");
  if (workers_a == 0 || workers_b == 0)
    throw ConfigError("both executors need at least one worker");
  if (!(slowdown_a >= 1.0) || !(slowdown_b >= 1.0))
    throw ConfigError("slowdown factors must be >= 1.0");
  if (emulated_fp64_slices < 0 || emulated_fp64_slices > 8)
    throw ConfigError("emulated_fp64_slices must be in [0, 8]");
  if (gpus < 1) throw ConfigError("gpus must be >= 1");
  if (comm < 0 || comm > 2) throw ConfigError("comm must be 0 (auto), 1 (NCCL) or 2 (in-process)");
}

Partition partition_for_fraction(double f, std::size_t rows) {
  std::size_t split = 0;
  check(hs_partition_for_fraction(f, rows, &split));
  return Partition{split, f};
}

std::size_t cholesky_border(double f, std::size_t column, std::size_t rows) {
  std::size_t beta = 0;
  const hs_status s = hs_cholesky_border(f, column, rows, &beta);
  if (s == HS_ERR_CONFIG && f >= 0.0 && f <= 1.0)
    throw std::out_of_range(hs_last_error());
  check(s);
  return beta;
}

CholeskyPlan CholeskyPlan::for_fraction(double f, std::size_t rows) {
  CholeskyPlan p;
  p.fraction = f;
  p.borders.resize(rows);
  for (std::size_t j = 0; j < rows; ++j) {
    p.borders[j] = cholesky_border(f, j, rows);
    if (j > 0 && p.borders[j] > p.borders[j - 1])
      p.shifts.push_back({j, p.borders[j] - p.borders[j - 1]});
  }
  return p;
}

std::size_t CholeskyPlan::blocks_on_b(std::size_t column) const {
  const std::size_t t = borders.size() - 1 - column;
  const std::size_t k = borders[column] - column;
  return (t * (t + 1) - (k - 1) * k) / 2;
}

std::size_t CholeskyPlan::trailing_blocks(std::size_t column, std::size_t rows) {
  const std::size_t t = rows - 1 - column;
  return t * (t + 1) / 2;
}

const char* to_string(TransferKind k) {
  static const char* names[] = {"scalar", "subvector", "block", "block_row",
                                "initial_matrix", "result"};
  return names[static_cast<int>(k)];
}
const char* to_string(Direction d) {
  static const char* names[] = {"a_to_b", "b_to_a", "bidirectional"};
  return names[static_cast<int>(d)];
}

std::uint64_t TransferLedger::total_bytes() const {
  std::uint64_t s = 0;
  for (const auto& e : entries_) s += e.bytes;
  return s;
}
std::uint64_t TransferLedger::bytes_of(TransferKind k) const {
  std::uint64_t s = 0;
  for (const auto& e : entries_) s += e.kind == k ? e.bytes : 0;
  return s;
}
std::size_t TransferLedger::count_of(TransferKind k) const {
  return (std::size_t)std::count_if(entries_.begin(), entries_.end(),
                                    [&](const TransferEntry& e) { return e.kind == k; });
}
std::size_t TransferLedger::count_of(TransferKind k, Direction d) const {
  return (std::size_t)std::count_if(
      entries_.begin(), entries_.end(),
      [&](const TransferEntry& e) { return e.kind == k && e.direction == d; });
}

// ---- runtime ---------------------------------------------------------------

Runtime::Runtime(std::size_t wa, std::size_t wb, double sa, double sb, bool audit)
    : audit_(audit) {
  if (wa == 0 || wb == 0) throw ConfigError("both executors need at least one worker");
  if (!(sa >= 1.0) || !(sb >= 1.0)) throw ConfigError("slowdown factors must be >= 1.0");
}

Runtime::Runtime(const SolverConfig& cfg)
    : device_(cfg.device), gpus_(cfg.gpus), comm_(cfg.comm) {
  cfg.validate();
}

// The reference builds a fresh Runtime per solve (bench.cpp:108); its
// state is the ledger, which a Runtime here still owns. The GPU contexts
// behind it (streams, cached device matrices, workspaces, NCCL
// communicators) are pooled per (device, gpus, comm) for the process, so
// repeated Runtimes do not pay device allocation and communicator setup on
// every solve. Solves are serial (SPEC: one solve at a time).
namespace {
struct Pooled {
  hs_ctx* ctx = nullptr;
  hs_group* group = nullptr;
};
std::mutex g_pool_mu;
std::map<std::tuple<int, int, int>, Pooled>& pool() {
  static auto* p = new std::map<std::tuple<int, int, int>, Pooled>;  // never destroyed
  return *p;
}
}  // namespace

Runtime::~Runtime() = default;

hs_group* Runtime::group() {
  if (gpus_ <= 1) return nullptr;
  if (!group_) {
    std::lock_guard<std::mutex> lk(g_pool_mu);
    Pooled& p = pool()[{device_, gpus_, comm_}];
    if (!p.group) {
      int count = 0;
      check(hs_device_count(&count));
      std::vector<int> dev(gpus_);
      for (int r = 0; r < gpus_; ++r) dev[r] = (device_ + r) % std::max(count, 1);
      check(hs_group_create(gpus_, dev.data(), comm_, &p.group));
    }
    group_ = p.group;
    ctx_ = hs_group_ctx(group_, 0);
    hs_ctx_ledger_clear(ctx_);  // a fresh Runtime starts with an empty ledger
  }
  return group_;
}

hs_ctx* Runtime::native() {
  if (gpus_ > 1) return (group(), ctx_);
  if (!ctx_) {
    std::lock_guard<std::mutex> lk(g_pool_mu);
    Pooled& p = pool()[{device_, 1, 0}];
    if (!p.ctx) check(hs_ctx_create(device_, nullptr, &p.ctx));
    ctx_ = p.ctx;
    hs_ctx_ledger_clear(ctx_);
  }
  return ctx_;
}

void Runtime::sync_ledger() {
  if (!ctx_) return;
  std::vector<hs_ledger_entry> e(hs_ctx_ledger_size(ctx_));
  e.resize(hs_ctx_ledger_read(ctx_, e.data(), e.size()));
  hs_ctx_ledger_clear(ctx_);
  for (const hs_ledger_entry& x : e)
    ledger_.append(TransferEntry{static_cast<TransferKind>(x.kind),
                                 static_cast<Direction>(x.direction), x.bytes, x.step});
}

// ---- assembly --------------------------------------------------------------

namespace rng {
std::uint64_t at(std::uint64_t key, std::uint64_t counter) {
  return hs_rng_at(key, counter);
}
double uniform01(std::uint64_t key, std::uint64_t counter) {
  return static_cast<double>(hs_rng_at(key, counter) >> 11) * 0x1.0p-53;
}
double uniform_pm1(std::uint64_t key, std::uint64_t counter) {
  return hs_rng_uniform_pm1(key, counter);
}
}  // namespace rng

std::vector<double> generate_inputs(std::size_t n, std::size_t dim,
                                    std::uint64_t seed) {
  std::vector<double> out(n * dim);
  check(hs_generate_inputs(n, dim, seed, out.data()));
  return out;
}

double median_pairwise_distance(const std::vector<double>& pts, std::size_t n,
                                std::size_t dim) {
  return hs_median_pairwise_distance(pts.data(), n, dim);
}

BlockedSPDMatrix generate_spd(std::size_t n, std::size_t b,
                              const KernelParams& p, std::uint64_t seed) {
  if (!(p.sigma_f2 > 0.0) || !(p.sigma_n2 > 0.0))
    throw ConfigError("kernel variances must be positive");
  BlockedSPDMatrix out(n, b);
  hs_matrix* m = nullptr;
  check(hs_matrix_create(default_ctx(), n, b, &m));
  hs_status s = hs_generate_spd(m, p.sigma_f2, p.length_scale, p.sigma_n2, p.dim, seed);
  if (s == HS_OK) s = hs_matrix_download(m, out.data());
  hs_matrix_destroy(m);
  check(s);
  return out;
}

BlockVector generate_rhs(std::size_t n, std::size_t b, std::uint64_t seed) {
  BlockVector v(n, b);
  check(hs_generate_rhs(n, b, seed, v.data()));
  return v;
}

// ---- solvers ---------------------------------------------------------------

CgResult solve_cg(const BlockedSPDMatrix& a, const BlockVector& rhs,
                  const SolverConfig& cfg, Runtime& rt) {
  cfg.validate();
  if (rhs.n() != a.n() || rhs.block_size() != a.block_size())
    throw ConfigError("matrix and right-hand side shapes do not match");
  CgResult res{BlockVector(a.n(), a.block_size()), CgStats{}};
  hs_cg_params p{cfg.eps, cfg.max_iters, cfg.recompute_interval,
                 cfg.record_trace ? 1 : 0};
  hs_cg_stats st{};
  std::vector<double> trace(cfg.record_trace ? 3 * std::max<std::size_t>(cfg.max_iters, 1) : 0);
  if (hs_group* g = rt.group()) {
    check(hs_group_set_row_fraction(g, cfg.fraction));
    check(hs_group_solve_cg_host(g, a.n(), a.block_size(), a.data(), rhs.data(), &p,
                                 res.x.data(), &st, cfg.record_trace ? trace.data() : nullptr));
  } else {
    check(hs_solve_cg_host(rt.native(), a.n(), a.block_size(), a.data(), rhs.data(), &p,
                           res.x.data(), &st, cfg.record_trace ? trace.data() : nullptr));
  }
  rt.add_transfer_ms(st.transfer_ms);
  rt.sync_ledger();
  res.stats.iterations = st.iterations;
  res.stats.recomputations = st.recomputations;
  res.stats.converged = st.converged != 0;
  res.stats.u0 = st.u0;
  res.stats.true_residual = st.true_residual;
  res.stats.wall_ms = st.wall_ms;
  res.stats.compute_ms = st.compute_ms;
  // the split that ran: rank 0's block rows with 2 GPUs (partition.hpp:8-18
  // semantics for B = rank 0), none on one GPU
  res.stats.partition = Partition{0, cfg.fraction};
  if (rt.gpus() == 2 && cfg.fraction > 0.0 && cfg.fraction < 1.0 && a.block_rows() >= 2)
    res.stats.partition.split_row =
        std::min(std::max<std::size_t>(partition_for_fraction(cfg.fraction, a.block_rows()).split_row, 1),
                 a.block_rows() - 1);
  for (std::size_t k = 0; cfg.record_trace && k < st.iterations; ++k)
    res.stats.trace.push_back({trace[3 * k], trace[3 * k + 1], trace[3 * k + 2]});
  return res;
}

FactorizeStats factorize(BlockedSPDMatrix& a, const SolverConfig& cfg, Runtime& rt) {
  cfg.validate();
  hs_chol_stats st{};
  if (hs_group* g = rt.group()) {
    check(hs_group_set_cholesky_gemm(g, cfg.emulated_fp64_slices));
    check(hs_group_factorize_host(g, a.n(), a.block_size(), a.data(), &st));
  } else {
    check(hs_ctx_set_cholesky_gemm(rt.native(), cfg.emulated_fp64_slices));
    check(hs_factorize_host(rt.native(), a.n(), a.block_size(), a.data(), &st));
  }
  rt.add_transfer_ms(st.transfer_ms);
  rt.sync_ledger();
  FactorizeStats out;
  out.plan = plan_for(cfg, a.block_rows());
  out.factor_ms = st.factor_ms;
  out.compute_ms = st.compute_ms;
  return out;
}

BlockVector forward_substitute(const BlockedSPDMatrix& l, const BlockVector& rhs) {
  if (rhs.n() != l.n() || rhs.block_size() != l.block_size())
    throw ConfigError("factor and right-hand side shapes do not match");
  BlockVector y(l.n(), l.block_size());
  check(hs_forward_substitute_host(default_ctx(), l.n(), l.block_size(), l.data(),
                                   rhs.data(), y.data()));
  return y;
}

BlockVector back_substitute(const BlockedSPDMatrix& l, const BlockVector& y) {
  if (y.n() != l.n() || y.block_size() != l.block_size())
    throw ConfigError("factor and right-hand side shapes do not match");
  BlockVector x(l.n(), l.block_size());
  check(hs_back_substitute_host(default_ctx(), l.n(), l.block_size(), l.data(),
                                y.data(), x.data()));
  return x;
}

SpdSolveResult solve_spd(BlockedSPDMatrix& a, const BlockVector& rhs,
                         const SolverConfig& cfg, Runtime& rt) {
  cfg.validate();
  if (rhs.n() != a.n() || rhs.block_size() != a.block_size())
    throw ConfigError("matrix and right-hand side shapes do not match");
  SpdSolveResult res{BlockVector(a.n(), a.block_size()), SpdSolveStats{}};
  hs_chol_stats st{};
  if (hs_group* g = rt.group()) {
    check(hs_group_set_cholesky_gemm(g, cfg.emulated_fp64_slices));
    check(hs_group_solve_spd_host(g, a.n(), a.block_size(), a.data(), rhs.data(),
                                  res.x.data(), &st));
  } else {
    check(hs_ctx_set_cholesky_gemm(rt.native(), cfg.emulated_fp64_slices));
    check(hs_solve_spd_host(rt.native(), a.n(), a.block_size(), a.data(), rhs.data(),
                            res.x.data(), &st));
  }
  rt.add_transfer_ms(st.transfer_ms);
  rt.sync_ledger();
  res.stats.plan = plan_for(cfg, a.block_rows());
  res.stats.factor_ms = st.factor_ms;
  res.stats.solve_ms = st.solve_ms;
  res.stats.wall_ms = st.wall_ms;
  res.stats.compute_ms = st.compute_ms;
  res.stats.true_residual = st.true_residual;
  return res;
}

}  // namespace hsolve
