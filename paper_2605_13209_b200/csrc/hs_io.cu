// BSPD1 matrix / vector files (reference matrix_io.hpp:9-19,
// matrix_io.cpp:70-139) — host-side format handling plus the B200 device
// path: files stream straight into (or out of) HBM tiles through a pinned
// staging ring, so a 68.8 GB n=131072 matrix never needs a host copy.
//
// Format: "BSPD", version byte 0x01, u64 n, u64 b (little endian), then the
// packed lower-triangular tiles in triangular order (tile (i, j) at
// (i(i+1)/2 + j) * b * b doubles), b*b FP64 little-endian values row-major
// per tile. Vector files: u64 n then n FP64 values. Error kinds as
// matrix_io.cpp: io (open/write), format (magic, implausible header),
// version_mismatch, truncated_file (expected vs actual byte counts).
#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "hs_internal.h"

static_assert(__BYTE_ORDER__ == __ORDER_LITTLE_ENDIAN__,
              "BSPD1 is little endian; this build assumes a little-endian host");

namespace hs {
namespace {

constexpr char kMagic[4] = {'B', 'S', 'P', 'D'};
constexpr unsigned char kVersion = 0x01;
constexpr uint64_t kHeader = 4 + 1 + 8 + 8;
constexpr uint64_t kMaxSide = 1ull << 32;   // header sanity caps
constexpr uint64_t kMaxBlock = 1ull << 20;
constexpr size_t kStage = 64ull << 20;      // bytes per staging buffer
constexpr int kStages = 3;

// RAII file descriptor.
struct Fd {
  int fd = -1;
  ~Fd() {
    if (fd >= 0) close(fd);
  }
};

void open_read(Fd& f, const char* path, uint64_t* size) {
  f.fd = open(path, O_RDONLY | O_CLOEXEC);
  if (f.fd < 0) throw Failure{HS_ERR_IO, std::string("cannot open ") + path};
  struct stat st;
  if (fstat(f.fd, &st) != 0)
    throw Failure{HS_ERR_IO, std::string("cannot stat ") + path};
  *size = (uint64_t)st.st_size;
}

void open_write(Fd& f, const char* path, bool truncate) {
  f.fd = open(path, O_WRONLY | O_CREAT | O_CLOEXEC | (truncate ? O_TRUNC : 0), 0644);
  if (f.fd < 0)
    throw Failure{HS_ERR_IO, std::string("cannot open ") + path + " for writing"};
}

// Full pread / pwrite (loops over short transfers).
bool pread_all(int fd, void* dst, size_t count, uint64_t off) {
  char* p = static_cast<char*>(dst);
  while (count > 0) {
    const ssize_t r = pread(fd, p, count, (off_t)off);
    if (r <= 0) return false;
    p += r;
    off += (uint64_t)r;
    count -= (size_t)r;
  }
  return true;
}

void pwrite_all(int fd, const void* src, size_t count, uint64_t off,
                const char* path) {
  const char* p = static_cast<const char*>(src);
  while (count > 0) {
    const ssize_t r = pwrite(fd, p, count, (off_t)off);
    if (r <= 0) throw Failure{HS_ERR_IO, std::string("write failed for ") + path};
    p += r;
    off += (uint64_t)r;
    count -= (size_t)r;
  }
}

uint64_t get_u64(const unsigned char* p) {
  uint64_t v;
  std::memcpy(&v, p, 8);
  return v;
}

// Header check in the reference's order (matrix_io.cpp:92-108): truncated
// header, magic, version, implausible n / b, then the payload length.
struct Header {
  uint64_t n, b, N, values;
};

Header read_header(int fd, uint64_t file_size, const char* path) {
  unsigned char h[kHeader] = {};
  const uint64_t got = std::min<uint64_t>(file_size, kHeader);
  if (!pread_all(fd, h, (size_t)got, 0))
    throw Failure{HS_ERR_IO, std::string("read failed for ") + path};
  // fields are checked as far as the bytes reach; a short header is
  // truncated at the first field it cuts
  auto short_header = [&] {
    return Failure{HS_ERR_TRUNCATED_FILE,
                   "file truncated: expected " + std::to_string(kHeader) +
                       " bytes, got " + std::to_string(got),
                   (int64_t)kHeader, (int64_t)got};
  };
  if (got < 4) throw short_header();
  if (std::memcmp(h, kMagic, 4) != 0)
    throw Failure{HS_ERR_FORMAT, std::string("bad magic in ") + path};
  if (got < 5) throw short_header();
  if (h[4] != kVersion)
    throw Failure{HS_ERR_VERSION_MISMATCH,
                  "unsupported file version " + std::to_string(h[4]) +
                      " (expected " + std::to_string(kVersion) + ")",
                  kVersion, h[4]};
  if (got < kHeader) throw short_header();
  Header r;
  r.n = get_u64(h + 5);
  r.b = get_u64(h + 13);
  if (r.n == 0 || r.b == 0 || r.n > kMaxSide || r.b > kMaxBlock)
    throw Failure{HS_ERR_FORMAT, "implausible header (n = " + std::to_string(r.n) +
                                     ", b = " + std::to_string(r.b) + ") in " + path};
  r.N = (r.n + r.b - 1) / r.b;
  // N (N + 1) / 2 * b^2 * 8 + header, every step overflow-checked: a header
  // whose size wraps 64 bits would otherwise pass the truncation check
  uint64_t tiles = 0, bb = 0, expected = 0;
  const bool wraps = __builtin_mul_overflow(r.N, r.N + 1, &tiles) ||
                     __builtin_mul_overflow(tiles / 2, 1, &tiles) ||
                     __builtin_mul_overflow(r.b, r.b, &bb) ||
                     __builtin_mul_overflow(tiles, bb, &r.values) ||
                     __builtin_mul_overflow(r.values, (uint64_t)8, &expected) ||
                     __builtin_add_overflow(expected, (uint64_t)kHeader, &expected);
  if (wraps)
    throw Failure{HS_ERR_FORMAT, "implausible header (n = " + std::to_string(r.n) +
                                     ", b = " + std::to_string(r.b) +
                                     ": size overflows 64 bits) in " + path};
  if (file_size < expected)
    throw Failure{HS_ERR_TRUNCATED_FILE,
                  "file truncated: expected " + std::to_string(expected) +
                      " bytes, got " + std::to_string(file_size),
                  (int64_t)expected, (int64_t)file_size};
  return r;
}

void write_header(int fd, uint64_t n, uint64_t b, const char* path) {
  unsigned char h[kHeader];
  std::memcpy(h, kMagic, 4);
  h[4] = kVersion;
  std::memcpy(h + 5, &n, 8);
  std::memcpy(h + 13, &b, 8);
  pwrite_all(fd, h, kHeader, 0, path);
}

// One contiguous piece of a transfer: `bytes` at file offset `off` <-> device
// address `dev`.
struct Piece {
  uint64_t off;
  char* dev;
  size_t bytes;
};

// The pieces of the rank's local tiles: one range for a row-sharded matrix
// (its block rows are contiguous in packed order), runs of consecutive owned
// tiles for a 2D block-cyclic one.
std::vector<Piece> pieces_of(const hs_matrix* m) {
  const size_t tb = m->b * m->b * sizeof(double);
  std::vector<Piece> out;
  if (m->layout == 0) {
    if (m->local_tiles())
      out.push_back({kHeader + (uint64_t)m->tile_lo * tb, (char*)m->d,
                     m->local_tiles() * tb});
    return out;
  }
  for (size_t k = 0; k < m->owned.size(); ++k) {
    const uint64_t off = kHeader + (uint64_t)m->owned[k] * tb;
    char* dev = (char*)m->d + k * tb;
    if (!out.empty() && out.back().off + out.back().bytes == off &&
        out.back().dev + out.back().bytes == dev)
      out.back().bytes += tb;
    else
      out.push_back({off, dev, tb});
  }
  return out;
}

// Pinned staging ring: while buffer k's H2D (or D2H) copy runs on the
// stream, the host fills (or drains) the next buffer with pread (pwrite).
struct Staging {
  char* buf[kStages] = {};
  cudaEvent_t ev[kStages] = {};
  bool busy[kStages] = {};
  Staging() {
    for (int k = 0; k < kStages; ++k) {
      HS_CUDA(cudaMallocHost(&buf[k], kStage));
      HS_CUDA(cudaEventCreateWithFlags(&ev[k], cudaEventDisableTiming));
    }
  }
  ~Staging() {
    for (int k = 0; k < kStages; ++k) {
      if (ev[k]) {
        cudaEventSynchronize(ev[k]);
        cudaEventDestroy(ev[k]);
      }
      if (buf[k]) cudaFreeHost(buf[k]);
    }
  }
  void wait(int k) {
    if (busy[k]) HS_CUDA(cudaEventSynchronize(ev[k]));
    busy[k] = false;
  }
};

void stream_in(hs_matrix* m, int fd, const char* path) {
  const std::vector<Piece> ps = pieces_of(m);
  cudaStream_t s = m->ctx->stream;
  Staging st;
  int k = 0;
  for (const Piece& p : ps) {
    for (size_t done = 0; done < p.bytes;) {
      const size_t len = std::min(kStage, p.bytes - done);
      st.wait(k);
      if (!pread_all(fd, st.buf[k], len, p.off + done))
        throw Failure{HS_ERR_IO, std::string("read failed for ") + path};
      HS_CUDA(cudaMemcpyAsync(p.dev + done, st.buf[k], len, cudaMemcpyHostToDevice, s));
      HS_CUDA(cudaEventRecord(st.ev[k], s));
      st.busy[k] = true;
      done += len;
      k = (k + 1) % kStages;
    }
  }
  HS_CUDA(cudaStreamSynchronize(s));
}

void stream_out(const hs_matrix* m, int fd, const char* path) {
  const std::vector<Piece> ps = pieces_of(m);
  cudaStream_t s = m->ctx->stream;
  Staging st;
  // chunk list, then a software pipeline: issue D2H of chunk q, write q-1
  struct Chunk {
    uint64_t off;
    const char* dev;
    size_t len;
  };
  std::vector<Chunk> cs;
  for (const Piece& p : ps)
    for (size_t d = 0; d < p.bytes; d += kStage)
      cs.push_back({p.off + d, p.dev + d, std::min(kStage, p.bytes - d)});
  const size_t q = cs.size();
  for (size_t i = 0; i < q + kStages - 1; ++i) {
    if (i < q) {
      const int k = (int)(i % kStages);
      HS_CUDA(cudaMemcpyAsync(st.buf[k], cs[i].dev, cs[i].len, cudaMemcpyDeviceToHost, s));
      HS_CUDA(cudaEventRecord(st.ev[k], s));
      st.busy[k] = true;
    }
    if (i + 1 >= kStages) {
      const size_t w = i + 1 - kStages;
      const int k = (int)(w % kStages);
      st.wait(k);
      pwrite_all(fd, st.buf[k], cs[w].len, cs[w].off, path);
    }
  }
}

}  // namespace
}  // namespace hs

using namespace hs;

#define HS_API_BEGIN \
  clear_error();     \
  try {
#define HS_API_END                                                         \
  return HS_OK;                                                            \
  }                                                                        \
  catch (const Failure& f) {                                               \
    set_error(f.status, f.msg, f.a, f.b);                                  \
    return f.status;                                                       \
  }                                                                        \
  catch (const std::exception& e) {                                        \
    set_error(HS_ERR_CUDA, e.what());                                      \
    return HS_ERR_CUDA;                                                    \
  }

extern "C" {

hs_status hs_bspd1_probe(const char* path, size_t* n, size_t* b) {
  HS_API_BEGIN
  HS_REQUIRE(path, HS_ERR_CONFIG, "null path");
  Fd f;
  uint64_t size = 0;
  open_read(f, path, &size);
  const Header h = read_header(f.fd, size, path);
  if (n) *n = (size_t)h.n;
  if (b) *b = (size_t)h.b;
  HS_API_END
}

hs_status hs_bspd1_read(const char* path, double* host, size_t count) {
  HS_API_BEGIN
  HS_REQUIRE(path && host, HS_ERR_CONFIG, "null pointer");
  Fd f;
  uint64_t size = 0;
  open_read(f, path, &size);
  const Header h = read_header(f.fd, size, path);
  HS_REQUIRE(count == h.values, HS_ERR_CONFIG,
             "destination holds " + std::to_string(count) + " values, file has " +
                 std::to_string(h.values));
  if (!pread_all(f.fd, host, h.values * 8, kHeader))
    throw Failure{HS_ERR_IO, std::string("read failed for ") + path};
  HS_API_END
}

hs_status hs_bspd1_write(const char* path, size_t n, size_t b, const double* host) {
  HS_API_BEGIN
  HS_REQUIRE(path && host && n > 0 && b > 0, HS_ERR_CONFIG, "bad arguments");
  const uint64_t N = (n + b - 1) / b;
  const uint64_t values = N * (N + 1) / 2 * b * b;
  Fd f;
  open_write(f, path, true);
  write_header(f.fd, n, b, path);
  pwrite_all(f.fd, host, values * 8, kHeader, path);
  HS_API_END
}

hs_status hs_vector_probe(const char* path, size_t* n) {
  HS_API_BEGIN
  HS_REQUIRE(path, HS_ERR_CONFIG, "null path");
  Fd f;
  uint64_t size = 0;
  open_read(f, path, &size);
  unsigned char h[8];
  if (size < 8 || !pread_all(f.fd, h, 8, 0))
    throw Failure{HS_ERR_TRUNCATED_FILE,
                  "file truncated: expected 8 bytes, got " + std::to_string(size), 8,
                  (int64_t)size};
  const uint64_t len = get_u64(h);
  if (len == 0 || len > kMaxSide)
    throw Failure{HS_ERR_FORMAT, "implausible vector length " + std::to_string(len) +
                                     " in " + path};
  if (size < 8 + len * 8)
    throw Failure{HS_ERR_TRUNCATED_FILE,
                  "file truncated: expected " + std::to_string(8 + len * 8) +
                      " bytes, got " + std::to_string(size),
                  (int64_t)(8 + len * 8), (int64_t)size};
  if (n) *n = (size_t)len;
  HS_API_END
}

hs_status hs_vector_read(const char* path, double* out, size_t n) {
  HS_API_BEGIN
  size_t len = 0;
  const hs_status s = hs_vector_probe(path, &len);
  if (s != HS_OK) {
    int64_t a, b;
    hs_last_error_payload(&a, &b);
    throw Failure{s, hs_last_error(), a, b};
  }
  HS_REQUIRE(out && n == len, HS_ERR_CONFIG, "vector length mismatch");
  Fd f;
  uint64_t size = 0;
  open_read(f, path, &size);
  if (!pread_all(f.fd, out, len * 8, 8))
    throw Failure{HS_ERR_IO, std::string("read failed for ") + path};
  HS_API_END
}

hs_status hs_vector_write(const char* path, size_t n, const double* v) {
  HS_API_BEGIN
  HS_REQUIRE(path && v && n > 0, HS_ERR_CONFIG, "bad arguments");
  Fd f;
  open_write(f, path, true);
  const uint64_t len = n;
  pwrite_all(f.fd, &len, 8, 0, path);
  pwrite_all(f.fd, v, n * 8, 8, path);
  HS_API_END
}

hs_status hs_matrix_load_bspd1(hs_ctx* c, const char* path, int cyclic,
                               hs_matrix** out) {
  HS_API_BEGIN
  HS_REQUIRE(c && path && out, HS_ERR_CONFIG, "null pointer");
  Fd f;
  uint64_t size = 0;
  open_read(f, path, &size);
  const Header h = read_header(f.fd, size, path);
  hs_matrix* m = nullptr;
  const hs_status s = cyclic ? hs_matrix_create_cyclic(c, h.n, h.b, &m)
                             : hs_matrix_create(c, h.n, h.b, &m);
  if (s != HS_OK) throw Failure{s, hs_last_error()};
  try {
    HS_CUDA(cudaSetDevice(c->device));
    stream_in(m, f.fd, path);
  } catch (...) {
    hs_matrix_destroy(m);
    throw;
  }
  m->has_inv = false;
  *out = m;
  HS_API_END
}

hs_status hs_matrix_save_bspd1(const hs_matrix* m, const char* path) {
  HS_API_BEGIN
  HS_REQUIRE(m && path, HS_ERR_CONFIG, "null pointer");
  const hs_ctx* c = m->ctx;
  HS_CUDA(cudaSetDevice(c->device));
  HS_CUDA(cudaStreamSynchronize(c->stream));
  Fd f;
  // a single rank owns the whole file and may truncate it; ranks of a
  // distributed matrix write disjoint ranges of a shared file
  open_write(f, path, c->world == 1);
  if (c->rank == 0) write_header(f.fd, m->n, m->b, path);
  stream_out(m, f.fd, path);
  const uint64_t total = kHeader + (uint64_t)tri((int64_t)m->N, 0) * m->b * m->b * 8;
  const bool last_owner = m->layout == 1 ? c->rank == c->world - 1 : m->row_hi == m->N;
  if (last_owner && ftruncate(f.fd, (off_t)total) != 0)
    throw Failure{HS_ERR_IO, std::string("cannot size ") + path};
  HS_API_END
}

}  // extern "C"
