// hsolve B200 host API (libhsolve_b200.so): the reference's C++ solver API,
// re-implemented over the sm_100a C ABI (hs_cuda.h).
//
// Reference headers this replaces (paths relative to /root/reference/proj):
//   blocked_matrix.hpp, solver_config.hpp, errors.hpp, partition.hpp,
//   transfer_ledger.hpp, executor.hpp (Runtime), genmat.hpp, cg_solver.hpp,
//   cholesky_solver.hpp; matrix_io.hpp and bench.hpp have their own headers
//   next to this one. The per-name headers next to this one include it,
//   so `#include "hsolve/cg_solver.hpp"` keeps compiling unchanged.
//
// Semantics kept: packed lower-triangular b x b tiles with identity padding,
// SolverConfig fields and validate(), exception types and ErrorKind names,
// NotConverged as a status, factorize() in place with stale diagonal-tile
// upper halves, solve_spd() destroying its matrix. Changed: arithmetic runs
// on B200s (Runtime = GPU context, or a group of `gpus` GPUs), `fraction`
// sets the CG row split of a 2-GPU Runtime, `workers_*` / `slowdown_*` are
// accepted but unused, and the transfer ledger holds the multi-GPU
// collectives (empty for one GPU, as in the reference's homogeneous modes).
#pragma once

#include <cstddef>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

struct hs_ctx;
struct hs_group;

namespace hsolve {

// ---- errors (errors.hpp:10-127) -------------------------------------------

enum class ErrorKind {
  config,
  not_spd,
  singular_block,
  numerical,
  not_converged,
  residency,
  format,
  version_mismatch,
  truncated_file,
  io,
};

const char* to_string(ErrorKind kind);

class Error : public std::runtime_error {
 public:
  Error(ErrorKind kind, const std::string& what)
      : std::runtime_error(what), kind_(kind) {}
  ErrorKind kind() const { return kind_; }

 private:
  ErrorKind kind_;
};

struct ConfigError : Error {
  explicit ConfigError(const std::string& m) : Error(ErrorKind::config, m) {}
};

class NotSpdError : public Error {
 public:
  NotSpdError(std::ptrdiff_t block_row, std::size_t pivot_index);
  std::ptrdiff_t block_row() const { return row_; }
  std::size_t pivot_index() const { return pivot_; }

 private:
  std::ptrdiff_t row_;
  std::size_t pivot_;
};

class SingularBlockError : public Error {
 public:
  explicit SingularBlockError(std::size_t diagonal_index);
  std::size_t diagonal_index() const { return index_; }

 private:
  std::size_t index_;
};

struct NumericalError : Error {
  explicit NumericalError(const std::string& m) : Error(ErrorKind::numerical, m) {}
};
struct ResidencyError : Error {
  explicit ResidencyError(const std::string& m) : Error(ErrorKind::residency, m) {}
};
struct FormatError : Error {
  explicit FormatError(const std::string& m) : Error(ErrorKind::format, m) {}
};
class VersionMismatchError : public Error {
 public:
  VersionMismatchError(unsigned expected, unsigned actual)
      : Error(ErrorKind::version_mismatch,
              "unsupported file version " + std::to_string(actual) +
                  " (expected " + std::to_string(expected) + ")") {}
};
class TruncatedFileError : public Error {
 public:
  TruncatedFileError(std::uint64_t expected_bytes, std::uint64_t actual_bytes)
      : Error(ErrorKind::truncated_file,
              "file truncated: expected " + std::to_string(expected_bytes) +
                  " bytes, got " + std::to_string(actual_bytes)),
        expected_(expected_bytes),
        actual_(actual_bytes) {}
  std::uint64_t expected_bytes() const { return expected_; }
  std::uint64_t actual_bytes() const { return actual_; }

 private:
  std::uint64_t expected_, actual_;
};
struct IoError : Error {
  explicit IoError(const std::string& m) : Error(ErrorKind::io, m) {}
};
// Device / runtime failure: no reference counterpart (a real GPU can fail).
struct DeviceError : Error {
  explicit DeviceError(const std::string& m) : Error(ErrorKind::io, m) {}
};

// ---- storage (blocked_matrix.hpp:10-89) ------------------------------------

std::size_t block_index(std::size_t i, std::size_t j, std::size_t block_rows);

class BlockedSPDMatrix {
 public:
  BlockedSPDMatrix(std::size_t n, std::size_t b);
  static BlockedSPDMatrix identity(std::size_t n, std::size_t b);

  std::size_t n() const { return n_; }
  std::size_t block_size() const { return b_; }
  std::size_t block_rows() const { return rows_; }
  std::size_t block_count() const { return rows_ * (rows_ + 1) / 2; }
  std::size_t padded_n() const { return rows_ * b_; }
  std::size_t pad() const { return padded_n() - n_; }

  double* block(std::size_t i, std::size_t j) {
    return v_.data() + block_index(i, j, rows_) * b_ * b_;
  }
  const double* block(std::size_t i, std::size_t j) const {
    return v_.data() + block_index(i, j, rows_) * b_ * b_;
  }
  double element(std::size_t p, std::size_t q) const;
  void set(std::size_t p, std::size_t q, double value);

  double* data() { return v_.data(); }
  const double* data() const { return v_.data(); }
  std::size_t value_count() const { return v_.size(); }
  void apply_identity_padding();

 private:
  std::size_t n_, b_, rows_;
  std::vector<double> v_;
};

class BlockVector {
 public:
  BlockVector(std::size_t n, std::size_t b);
  std::size_t n() const { return n_; }
  std::size_t block_size() const { return b_; }
  std::size_t block_rows() const { return rows_; }
  std::size_t padded_n() const { return rows_ * b_; }
  double* row(std::size_t i) { return v_.data() + i * b_; }
  const double* row(std::size_t i) const { return v_.data() + i * b_; }
  double& operator[](std::size_t i) { return v_[i]; }
  double operator[](std::size_t i) const { return v_[i]; }
  double* data() { return v_.data(); }
  const double* data() const { return v_.data(); }

 private:
  std::size_t n_, b_, rows_;
  std::vector<double> v_;
};

// ---- configuration (solver_config.hpp:12-26) -------------------------------

struct SolverConfig {
  double eps = 1e-6;
  std::size_t max_iters = 500;
  std::size_t recompute_interval = 50;
  double fraction = 0.0;
  std::size_t block_size = 32;
  std::size_t workers_a = 2;
  std::size_t workers_b = 2;
  double slowdown_a = 1.0;
  double slowdown_b = 1.0;
  std::uint64_t seed = 42;
  bool record_trace = false;
  int device = 0;  // B200 build: GPU ordinal of the Runtime (rank 0's)
  // B200 build: GPUs the work is partitioned over (the reference's two
  // executors generalised to G devices of one process). CG shards block rows
  // (with G == 2, `fraction` in (0, 1) gives rank 0 the reference's
  // partition_for_fraction share, partition.cpp:11-22); Cholesky uses a 2D
  // block-cyclic tile grid. Rank r runs on device (device + r) % count.
  int gpus = 1;
  // B200 build: collectives of a multi-GPU Runtime. 0 = auto (NCCL when every
  // rank has its own device, else in-process), 1 = NCCL, 2 = in-process
  // device copies (ranks may share a GPU).
  int comm = 0;
  // B200 build: Cholesky trailing-update engine. 0 = FP64 DMMA tensor cores
  // (the reference's arithmetic); 1..8 = FP64 emulated on the INT8 tensor
  // cores with that many slices (8: FP64-level error bound).
  int emulated_fp64_slices = 0;
  void validate() const;
};

// ---- work split (partition.hpp:8-47) ---------------------------------------

struct Partition {
  std::size_t split_row = 0;
  double fraction = 0.0;
};
Partition partition_for_fraction(double fraction, std::size_t block_rows);
std::size_t cholesky_border(double fraction, std::size_t column,
                            std::size_t block_rows);

struct ShiftEvent {
  std::size_t column = 0;
  std::size_t rows_moved = 0;
};

struct CholeskyPlan {
  double fraction = 0.0;
  std::vector<std::size_t> borders;
  std::vector<ShiftEvent> shifts;
  static CholeskyPlan for_fraction(double fraction, std::size_t block_rows);
  std::size_t blocks_on_b(std::size_t column) const;
  static std::size_t trailing_blocks(std::size_t column, std::size_t block_rows);
};

// ---- communication ledger (transfer_ledger.hpp:9-52) -----------------------

enum class TransferKind : std::uint8_t {
  scalar,
  subvector,
  block,
  block_row,
  initial_matrix,
  result
};
enum class Direction : std::uint8_t { a_to_b, b_to_a, bidirectional };
const char* to_string(TransferKind kind);
const char* to_string(Direction direction);

struct TransferEntry {
  TransferKind kind;
  Direction direction;
  std::uint64_t bytes;
  std::int64_t step;
};

class TransferLedger {
 public:
  void append(const TransferEntry& e) { entries_.push_back(e); }
  const std::vector<TransferEntry>& entries() const { return entries_; }
  std::size_t size() const { return entries_.size(); }
  std::uint64_t total_bytes() const;
  std::uint64_t bytes_of(TransferKind kind) const;
  std::size_t count_of(TransferKind kind) const;
  std::size_t count_of(TransferKind kind, Direction direction) const;
  void clear() { entries_.clear(); }

 private:
  std::vector<TransferEntry> entries_;
};

// ---- runtime = one GPU context (executor.hpp:128-221) ----------------------

class Runtime {
 public:
  // Reference signature; worker counts / slowdowns are validated, not used.
  Runtime(std::size_t workers_a, std::size_t workers_b, double slowdown_a,
          double slowdown_b, bool audit = true);
  explicit Runtime(const SolverConfig& cfg);
  ~Runtime();
  Runtime(const Runtime&) = delete;
  Runtime& operator=(const Runtime&) = delete;

  TransferLedger& ledger() { return ledger_; }
  const TransferLedger& ledger() const { return ledger_; }
  double transfer_seconds() const { return transfer_seconds_; }
  std::uint64_t observed_transfer_bytes() const { return 0; }
  bool audit() const { return audit_; }

  hs_ctx* native();  // the C-ABI context (rank 0's with gpus > 1)
  hs_group* group();  // the multi-GPU group (nullptr when gpus == 1)
  int gpus() const { return gpus_; }
  void add_transfer_ms(double ms) { transfer_seconds_ += ms * 1e-3; }
  // Moves the context's NCCL ledger entries (one per collective) into
  // ledger(); called by the solvers after each native call.
  void sync_ledger();

 private:
  int device_ = 0;
  int gpus_ = 1;
  int comm_ = 0;
  hs_ctx* ctx_ = nullptr;
  hs_group* group_ = nullptr;
  TransferLedger ledger_;
  double transfer_seconds_ = 0.0;
  bool audit_ = true;
};

// ---- assembly (genmat.hpp:14-45) -------------------------------------------

struct KernelParams {
  double sigma_f2 = 1.0;
  double length_scale = 0.0;
  double sigma_n2 = 1e-2;
  std::size_t dim = 2;
};

namespace rng {
std::uint64_t at(std::uint64_t key, std::uint64_t counter);
double uniform01(std::uint64_t key, std::uint64_t counter);
double uniform_pm1(std::uint64_t key, std::uint64_t counter);
}  // namespace rng

std::vector<double> generate_inputs(std::size_t n, std::size_t dim,
                                    std::uint64_t seed);
double median_pairwise_distance(const std::vector<double>& points,
                                std::size_t n, std::size_t dim);
// Tiles are assembled on the GPU and copied into host storage.
BlockedSPDMatrix generate_spd(std::size_t n, std::size_t b,
                              const KernelParams& params, std::uint64_t seed);
BlockVector generate_rhs(std::size_t n, std::size_t b, std::uint64_t seed);

// ---- CG (cg_solver.hpp:13-49) ----------------------------------------------

struct CgIteration {
  double u;
  double alpha;
  double beta;
};

struct CgStats {
  std::size_t iterations = 0;
  std::size_t recomputations = 0;
  bool converged = false;
  double u0 = 0.0;
  double true_residual = 0.0;
  double wall_ms = 0.0;
  double compute_ms = 0.0;
  Partition partition;
  std::vector<CgIteration> trace;
};

struct CgResult {
  BlockVector x;
  CgStats stats;
};

CgResult solve_cg(const BlockedSPDMatrix& a, const BlockVector& rhs,
                  const SolverConfig& cfg, Runtime& rt);

// ---- Cholesky (cholesky_solver.hpp:12-58) ----------------------------------

struct FactorizeStats {
  CholeskyPlan plan;
  double factor_ms = 0.0;
  double compute_ms = 0.0;
};

struct SpdSolveStats {
  CholeskyPlan plan;
  double factor_ms = 0.0;
  double solve_ms = 0.0;
  double wall_ms = 0.0;
  double compute_ms = 0.0;
  double true_residual = 0.0;
};

struct SpdSolveResult {
  BlockVector x;
  SpdSolveStats stats;
};

FactorizeStats factorize(BlockedSPDMatrix& a, const SolverConfig& cfg,
                         Runtime& rt);
BlockVector forward_substitute(const BlockedSPDMatrix& l,
                               const BlockVector& rhs);
BlockVector back_substitute(const BlockedSPDMatrix& l, const BlockVector& y);
SpdSolveResult solve_spd(BlockedSPDMatrix& a, const BlockVector& rhs,
                         const SolverConfig& cfg, Runtime& rt);

}  // namespace hsolve
