// hsolve::save_matrix / load_matrix / save_vector / load_vector
// (reference matrix_io.hpp:9-19) over the C ABI's BSPD1 code (hs_io.cu), so
// the host API and the device streaming loader share one format
// implementation and one set of error kinds.
#include "hsolve/matrix_io.hpp"

#include "host_internal.hpp"

namespace hsolve {

using detail::check;

void save_matrix(const BlockedSPDMatrix& m, const std::string& path) {
  check(hs_bspd1_write(path.c_str(), m.n(), m.block_size(), m.data()));
}

BlockedSPDMatrix load_matrix(const std::string& path) {
  std::size_t n = 0, b = 0;
  check(hs_bspd1_probe(path.c_str(), &n, &b));
  BlockedSPDMatrix m(n, b);
  check(hs_bspd1_read(path.c_str(), m.data(), m.value_count()));
  return m;
}

void save_vector(const BlockVector& v, const std::string& path) {
  check(hs_vector_write(path.c_str(), v.n(), v.data()));
}

BlockVector load_vector(const std::string& path, std::size_t block_size) {
  std::size_t n = 0;
  check(hs_vector_probe(path.c_str(), &n));
  BlockVector v(n, block_size);
  check(hs_vector_read(path.c_str(), v.data(), n));
  return v;
}

}  // namespace hsolve
