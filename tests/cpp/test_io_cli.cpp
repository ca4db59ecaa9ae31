// Drop-in check of matrix_io.hpp and bench.hpp (libhsolve_b200.so) with
// reference-style caller code (after proj/tests/test_genmat.cpp:98-175 and
// test_cli.cpp). `test_io_cli` runs the host-only part (no GPU: file format,
// error kinds, usage errors); `test_io_cli --gpu` adds gen / solve / sweep.
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <iterator>
#include <random>
#include <string>
#include <vector>

#include "hsolve/bench.hpp"
#include "hsolve/errors.hpp"
#include "hsolve/matrix_io.hpp"

using namespace hsolve;

static int failures = 0;
#define CHECK(c)                                               \
  do {                                                         \
    if (!(c)) {                                                \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #c); \
      ++failures;                                              \
    }                                                          \
  } while (0)

template <class E, class F>
static bool throws_as(F f) {
  try {
    f();
  } catch (const E&) {
    return true;
  } catch (...) {
    return false;
  }
  return false;
}

static std::vector<char> slurp(const std::string& p) {
  std::ifstream in(p, std::ios::binary);
  return {std::istreambuf_iterator<char>(in), {}};
}
static void spit(const std::string& p, const std::vector<char>& d) {
  std::ofstream out(p, std::ios::binary | std::ios::trunc);
  out.write(d.data(), (std::streamsize)d.size());
}

static int run_cli(const std::vector<std::string>& args) {
  std::vector<const char*> argv{"hsolve_bench"};
  for (const auto& a : args) argv.push_back(a.c_str());
  return bench::cli_main((int)argv.size(), argv.data());
}

static BlockedSPDMatrix filled(std::size_t n, std::size_t b, unsigned seed) {
  BlockedSPDMatrix m(n, b);
  std::mt19937_64 g(seed);
  std::uniform_real_distribution<double> u(-1.0, 1.0);
  for (std::size_t i = 0; i < m.value_count(); ++i) m.data()[i] = u(g);
  return m;
}

int main(int argc, char** argv) {
  const bool gpu = argc > 1 && std::string(argv[1]) == "--gpu";
  const std::string path = "/tmp/hsolve_b200_io.bspd";

  {  // round trip is bit-identical (test_genmat.cpp:98-114)
    std::mt19937_64 seeds(1234);
    for (int trial = 0; trial < 5; ++trial) {
      const std::size_t n = 16 + seeds() % 60, b = 1 + seeds() % 12;
      const BlockedSPDMatrix m = filled(n, b, (unsigned)seeds());
      save_matrix(m, path);
      const BlockedSPDMatrix back = load_matrix(path);
      CHECK(back.n() == n && back.block_size() == b);
      CHECK(std::memcmp(back.data(), m.data(), m.value_count() * 8) == 0);
    }
  }
  {  // error kinds (test_genmat.cpp:115-158)
    save_matrix(filled(20, 4, 3), path);
    const std::vector<char> good = slurp(path);
    std::vector<char> bad = good;
    bad[0] = 'X';
    spit(path, bad);
    CHECK(throws_as<FormatError>([&] { load_matrix(path); }));
    bad = good;
    bad[4] = 0x02;
    spit(path, bad);
    CHECK(throws_as<VersionMismatchError>([&] { load_matrix(path); }));
    bad = good;
    bad.resize(bad.size() - 100);
    spit(path, bad);
    try {
      load_matrix(path);
      CHECK(false);
    } catch (const TruncatedFileError& e) {
      CHECK(e.expected_bytes() == good.size());
      CHECK(e.actual_bytes() == good.size() - 100);
    }
    bad = good;
    bad.resize(10);
    spit(path, bad);
    CHECK(throws_as<TruncatedFileError>([&] { load_matrix(path); }));
    bad = good;
    for (int i = 0; i < 8; ++i) bad[5 + i] = (char)0xFF;
    spit(path, bad);
    CHECK(throws_as<FormatError>([&] { load_matrix(path); }));
    CHECK(throws_as<IoError>([] { load_matrix("/tmp/hsolve_does_not_exist.bspd"); }));
  }
  {  // vector round trip (test_genmat.cpp:165-175)
    BlockVector v(33, 8);
    for (std::size_t i = 0; i < 33; ++i) v[i] = 0.5 * (double)i - 3.0;
    save_vector(v, path);
    const BlockVector back = load_vector(path, 8);
    CHECK(back.n() == 33 && std::memcmp(back.data(), v.data(), v.padded_n() * 8) == 0);
  }
  {  // usage errors exit 2 (test_cli.cpp:54-63)
    CHECK(run_cli({"solve", "cg", "--size", "64", "--fraction", "1.5"}) == 2);
    CHECK(run_cli({"solve", "banana", "--size", "64"}) == 2);
    CHECK(run_cli({"solve", "cg"}) == 2);
    CHECK(run_cli({"nonsense"}) == 2);
    CHECK(run_cli({"sweep", "--sizes", "64", "--fractions", ""}) == 2);
    CHECK(run_cli({"sweep", "--sizes", "64", "--fractions", "zero"}) == 2);
    CHECK(run_cli({"sweep", "--sizes", "x,y", "--fractions", "0.5"}) == 2);
    CHECK(run_cli({"gen", "--size", "32"}) == 2);
  }
  if (gpu) {
    const std::string out = "/tmp/hsolve_b200_cli.csv";
    CHECK(run_cli({"gen", "--size", "48", "--block-size", "8", "--seed", "7", "--output",
                   path}) == 0);
    const BlockedSPDMatrix m = load_matrix(path);
    CHECK(m.n() == 48 && m.block_size() == 8);
    CHECK(run_cli({"solve", "cholesky", "--matrix", path, "--reps", "1", "--output", out}) ==
          0);
    bench::RunSpec rs;
    rs.algo = bench::Algo::cg;
    rs.n = 256;
    rs.cfg.block_size = 64;
    rs.reps = 2;
    const bench::Row r = bench::run_single(rs);
    CHECK(r.status == "converged" && r.iters > 0 && r.bytes_total == 0);
    CHECK(r.runtime_ms_median > 0.0 && r.iters_per_s > 0.0);
    const std::string line = bench::to_csv(r), head = bench::csv_header();
    CHECK(head.rfind("algo,n,block_size,fraction,", 0) == 0);
    CHECK(std::count(line.begin(), line.end(), ',') == std::count(head.begin(), head.end(), ','));
    std::remove(out.c_str());
  }
  std::remove(path.c_str());
  if (failures == 0) std::printf("ALL PASSED\n");
  return failures == 0 ? 0 : 1;
}
