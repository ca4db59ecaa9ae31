// Context, errors, host-side generators, work split, device matrices and the
// GP squared-exponential tile assembly kernel.
#include <dlfcn.h>
#include <math.h>
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "hs_internal.h"

namespace hs {

// ---------------------------------------------------------------------------
// errors

namespace {
thread_local std::string g_msg;
thread_local int64_t g_pa = -1, g_pb = -1;
}  // namespace

void set_error(int status, const std::string& msg, int64_t a, int64_t b) {
  (void)status;
  g_msg = msg;
  g_pa = a;
  g_pb = b;
}
void clear_error() {
  g_msg.clear();
  g_pa = g_pb = -1;
}

void launch_count(hs_ctx* c, int k) { c->launches += (uint64_t)k; }

// ---------------------------------------------------------------------------
// NCCL, resolved at run time so single-GPU users never need it.

struct Nccl {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*);
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int);
  ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*);
  ncclResult_t (*CommDestroy)(ncclComm_t);
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t,
                            ncclComm_t, cudaStream_t);
  ncclResult_t (*ReduceScatter)(const void*, void*, size_t, ncclDataType_t,
                                ncclRedOp_t, ncclComm_t, cudaStream_t);
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t,
                            ncclRedOp_t, ncclComm_t, cudaStream_t);
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int,
                            ncclComm_t, cudaStream_t);
  ncclResult_t (*GroupStart)();
  ncclResult_t (*GroupEnd)();
  const char* (*GetErrorString)(ncclResult_t);
};

static Nccl* load_nccl() {
  static Nccl* g = nullptr;
  if (g) return g;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  HS_REQUIRE(h, HS_ERR_CUDA, std::string("cannot load NCCL: ") + dlerror());
  Nccl* n = new Nccl;
  n->h = h;
#define HS_SYM(field, name)                                                 \
  n->field = reinterpret_cast<decltype(n->field)>(dlsym(h, name));          \
  HS_REQUIRE(n->field, HS_ERR_CUDA, "NCCL symbol missing: " name);
  HS_SYM(GetUniqueId, "ncclGetUniqueId");
  HS_SYM(CommInitRank, "ncclCommInitRank");
  HS_SYM(CommInitAll, "ncclCommInitAll");
  HS_SYM(CommDestroy, "ncclCommDestroy");
  HS_SYM(AllGather, "ncclAllGather");
  HS_SYM(ReduceScatter, "ncclReduceScatter");
  HS_SYM(AllReduce, "ncclAllReduce");
  HS_SYM(Broadcast, "ncclBroadcast");
  HS_SYM(GroupStart, "ncclGroupStart");
  HS_SYM(GroupEnd, "ncclGroupEnd");
  HS_SYM(GetErrorString, "ncclGetErrorString");
#undef HS_SYM
  g = n;
  return g;
}

void nccl_check(Nccl* n, ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    throw Failure{HS_ERR_CUDA, std::string(what) + ": " + n->GetErrorString(r)};
}

static void ledger_add(hs_ctx* c, LedgerKind kind, uint64_t bytes) {
  c->ledger.push_back(hs_ledger_entry{(uint8_t)kind, 2 /* bidirectional */,
                                      bytes, c->step});
}

static void custom_check(int r, const char* what) {
  if (r != 0) throw Failure{HS_ERR_CUDA, std::string(what) + ": custom transport failed"};
}

void comm_allgather(hs_ctx* c, const double* send, double* recv,
                    size_t count, LedgerKind kind) {
  if (c->local) {
    local_allgather(c, send, recv, count, c->stream);
    ledger_add(c, kind, (uint64_t)count * c->world * sizeof(double));
    return;
  }
  if (c->custom) {
    HS_CUDA(cudaStreamSynchronize(c->stream));
    custom_check(c->ops.allgather(c->ops.user, send, recv, count), "allgather");
    ledger_add(c, kind, (uint64_t)count * c->world * sizeof(double));
    return;
  }
  nccl_check(c->nccl,
             c->nccl->AllGather(send, recv, count, ncclFloat64,
                                (ncclComm_t)c->comm, c->stream),
             "ncclAllGather");
  ledger_add(c, kind, (uint64_t)count * c->world * sizeof(double));
}
void comm_reduce_scatter(hs_ctx* c, const double* send, double* recv,
                         size_t count, LedgerKind kind) {
  if (c->local) {
    local_reduce_scatter(c, send, recv, count, c->stream);
    ledger_add(c, kind, (uint64_t)count * sizeof(double));
    return;
  }
  if (c->custom) {
    HS_CUDA(cudaStreamSynchronize(c->stream));
    custom_check(c->ops.reduce_scatter(c->ops.user, send, recv, count), "reduce_scatter");
    ledger_add(c, kind, (uint64_t)count * sizeof(double));
    return;
  }
  nccl_check(c->nccl,
             c->nccl->ReduceScatter(send, recv, count, ncclFloat64, ncclSum,
                                    (ncclComm_t)c->comm, c->stream),
             "ncclReduceScatter");
  ledger_add(c, kind, (uint64_t)count * sizeof(double));
}
// broadcast from root's `send` into every rank's `recv` on stream s
void comm_bcast_on(hs_ctx* c, const double* send, double* recv, size_t count,
                   int root, cudaStream_t s, LedgerKind kind) {
  if (c->local) {
    local_bcast(c, send, recv, count, root, s);
    ledger_add(c, kind, (uint64_t)count * sizeof(double));
    return;
  }
  if (c->custom) {
    HS_CUDA(cudaStreamSynchronize(s));
    custom_check(c->ops.broadcast(c->ops.user, send, recv, count, root), "broadcast");
    ledger_add(c, kind, (uint64_t)count * sizeof(double));
    return;
  }
  nccl_check(c->nccl,
             c->nccl->Broadcast(send, recv, count, ncclFloat64, root,
                                (ncclComm_t)c->comm, s),
             "ncclBroadcast");
  ledger_add(c, kind, (uint64_t)count * sizeof(double));
}
void comm_group(hs_ctx* c, bool start) {
  if (c->custom || c->local) return;  // these collectives complete one by one
  nccl_check(c->nccl, start ? c->nccl->GroupStart() : c->nccl->GroupEnd(),
             "ncclGroupStart/End");
}
// element-wise max over ranks of `count` int64 values (in place)
void comm_allreduce_max_i64(hs_ctx* c, int64_t* buf, size_t count,
                            cudaStream_t s) {
  if (c->local) {
    local_allreduce_max_i64(c, buf, count, s);
    ledger_add(c, LK_SCALAR, (uint64_t)count * sizeof(int64_t));
    return;
  }
  if (c->custom) {
    HS_CUDA(cudaStreamSynchronize(s));
    custom_check(c->ops.allreduce_max_i64(c->ops.user, buf, count), "allreduce_max");
    ledger_add(c, LK_SCALAR, (uint64_t)count * sizeof(int64_t));
    return;
  }
  nccl_check(c->nccl,
             c->nccl->AllReduce(buf, buf, count, ncclInt64, ncclMax,
                                (ncclComm_t)c->comm, s),
             "ncclAllReduce");
  ledger_add(c, LK_SCALAR, (uint64_t)count * sizeof(int64_t));
}

// ---------------------------------------------------------------------------
// host generators — genmat.cpp:16-34, 45-54, 77-112, 156-162 (exact)

static uint64_t mix(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
static uint64_t rng_at(uint64_t key, uint64_t counter) {
  return mix(key ^ mix(counter));
}
static double uniform_pm1(uint64_t key, uint64_t counter) {
  return 2.0 * ((double)(rng_at(key, counter) >> 11) * 0x1.0p-53) - 1.0;
}
static const uint64_t kPointsStream = 0x706f696e74730001ull;
static const uint64_t kRhsStream = 0x7268730000000001ull;

static void gen_inputs(size_t n, size_t dim, uint64_t seed, double* out) {
  for (size_t i = 0; i < n; ++i) {
    const double t = (double)i * 0.01;
    for (size_t k = 0; k < dim; ++k) {
      double v = t;
      if (k != 0) {
        const double omega = 1.0 + 0.5 * (double)(k - 1);
        const double noise =
            0.05 * uniform_pm1(seed ^ kPointsStream, (uint64_t)i * dim + k);
        v = sin(omega * t) + noise;
      }
      out[i * dim + k] = v;
    }
  }
}

static double median_dist(const double* pts, size_t n, size_t dim) {
  const size_t m = std::min<size_t>(n, 512);
  if (m < 2) return 1.0;
  std::vector<double> d;
  d.reserve(m * (m - 1) / 2);
  for (size_t i = 0; i < m; ++i) {
    const size_t pi = i * n / m;
    for (size_t j = i + 1; j < m; ++j) {
      const size_t pj = j * n / m;
      double d2 = 0.0;
      for (size_t k = 0; k < dim; ++k) {
        const double e = pts[pi * dim + k] - pts[pj * dim + k];
        d2 += e * e;
      }
      d.push_back(sqrt(d2));
    }
  }
  auto mid = d.begin() + (std::ptrdiff_t)(d.size() / 2);
  std::nth_element(d.begin(), mid, d.end());
  return *mid == 0.0 ? 1.0 : *mid;
}

// ---------------------------------------------------------------------------
// work split

// Contiguous block-row ranges balanced by packed tile count (row i holds
// i+1 tiles): bounds[g] = first row with tri(row,0) >= g*T/G.
static std::vector<int64_t> row_bounds(int64_t N, int world) {
  std::vector<int64_t> b(world + 1, 0);
  const int64_t T = N * (N + 1) / 2;
  for (int g = 1; g < world; ++g) {
    const int64_t target = (T * g + world / 2) / world;
    int64_t r = b[g - 1];
    while (r < N && tri(r, 0) + (r + 1) / 2 < target) ++r;
    b[g] = r;
  }
  b[world] = N;
  return b;
}

// ---------------------------------------------------------------------------
// GP squared-exponential tile assembly (genmat.cpp:128-152).
// One CTA per (local tile, row chunk); consecutive threads write consecutive
// elements of a row (coalesced 8-B stores, one HBM write of the packed
// array). d2 uses explicit round-to-nearest mul/add (no FMA contraction) to
// keep the reference's rounding; exp is CUDA's double exp (<= 1 ulp).

template <int DIM>  // DIM > 0: compile-time dimension; 0: runtime `dim`
__global__ void __launch_bounds__(256)
    assemble_se_kernel(double* __restrict__ tiles, int64_t tile_base,
                       const int64_t* __restrict__ owned, int64_t n,
                       int b, const double* __restrict__ pts, int dim,
                       double sf2, double inv2l2, double sn2,
                       int rows_per_cta) {
  const int64_t t = owned ? owned[blockIdx.x] : tile_base + blockIdx.x;
  const int64_t i = tile_row(t);
  const int64_t j = t - tri(i, 0);
  const int r0 = blockIdx.y * rows_per_cta;
  const int r1 = min(b, r0 + rows_per_cta);
  double* blk = tiles + (int64_t)blockIdx.x * b * b;
  const double diag = __dadd_rn(sf2, sn2);
  // each thread owns column c: its point stays in registers; the row point
  // is warp-uniform (broadcast load); stores are coalesced along the row.
  // Interior tiles (off-diagonal, no padding) take a branch-free path with
  // four rows per iteration, so the exp constants and the address math are
  // shared by four independent exp evaluations.
  const bool interior = (i != j) && ((i + 1) * (int64_t)b <= n) && DIM > 0;
  for (int c = threadIdx.x; c < b; c += blockDim.x) {
    const int64_t q = j * b + c;
    double xq[DIM > 0 ? DIM : 1];
    if (DIM > 0 && q < n) {
#pragma unroll
      for (int k = 0; k < (DIM > 0 ? DIM : 1); ++k) xq[k] = __ldg(pts + q * DIM + k);
    }
    if (interior) {
      const double nl = -inv2l2;
      const double* prow = pts + (i * b + r0) * DIM;
      double* out = blk + (int64_t)r0 * b + c;
      int r = r0;
      for (; r + 4 <= r1; r += 4, prow += 4 * DIM, out += 4 * (int64_t)b) {
        double v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          double d2 = 0.0;
#pragma unroll
          for (int k = 0; k < (DIM > 0 ? DIM : 1); ++k) {
            const double d = __dsub_rn(__ldg(prow + u * DIM + k), xq[k]);
            d2 = __dadd_rn(d2, __dmul_rn(d, d));
          }
          v[u] = __dmul_rn(sf2, exp(__dmul_rn(d2, nl)));
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) __stcs(out + u * (int64_t)b, v[u]);
      }
      for (; r < r1; ++r, prow += DIM, out += b) {
        double d2 = 0.0;
#pragma unroll
        for (int k = 0; k < (DIM > 0 ? DIM : 1); ++k) {
          const double d = __dsub_rn(__ldg(prow + k), xq[k]);
          d2 = __dadd_rn(d2, __dmul_rn(d, d));
        }
        __stcs(out, __dmul_rn(sf2, exp(__dmul_rn(d2, nl))));
      }
      continue;
    }
    for (int r = r0; r < r1; ++r) {
      const int64_t p = i * b + r;
      double v;
      if (p >= n || q >= n) {
        v = (p == q) ? 1.0 : 0.0;
      } else if (p == q) {
        v = diag;
      } else {
        double d2 = 0.0;
        if (DIM > 0) {
#pragma unroll
          for (int k = 0; k < (DIM > 0 ? DIM : 1); ++k) {
            const double d = __dsub_rn(__ldg(pts + p * DIM + k), xq[k]);
            d2 = __dadd_rn(d2, __dmul_rn(d, d));
          }
        } else {
          for (int k = 0; k < dim; ++k) {
            const double d = __dsub_rn(__ldg(pts + p * dim + k), __ldg(pts + q * dim + k));
            d2 = __dadd_rn(d2, __dmul_rn(d, d));
          }
        }
        v = __dmul_rn(sf2, exp(__dmul_rn(-d2, inv2l2)));
      }
      __stcs(blk + (int64_t)r * b + c, v);
    }
  }
}

// identity padding of an uploaded/zeroed matrix's last block row
// (blocked_matrix.cpp:57-74)
__global__ void identity_pad_kernel(double* tiles, int64_t tile_base,
                                    const int64_t* lpos, int64_t n, int b,
                                    int64_t N) {
  const int64_t last = N - 1;
  const int64_t t = tri(last, 0) + blockIdx.x;  // tile (last, j)
  const int64_t j = blockIdx.x;
  const int64_t slot = lpos ? lpos[j] : t - tile_base;
  if (slot < 0) return;  // not on this rank
  double* blk = tiles + slot * b * b;
  for (int idx = threadIdx.x; idx < b * b; idx += blockDim.x) {
    const int r = idx / b, c = idx % b;
    const int64_t p = last * b + r, q = j * b + c;
    if (p < n) continue;
    blk[idx] = (p == q) ? 1.0 : 0.0;
  }
}

__global__ void fill_kernel(double* p, double v, int64_t count) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < count;
       k += (int64_t)gridDim.x * blockDim.x)
    p[k] = v;
}

void launch_fill(hs_ctx* c, double* p, double v, int64_t count) {
  if (count <= 0) return;
  const int grid = (int)std::min<int64_t>(ceil_div(count, 256), 4 * 148);
  fill_kernel<<<grid, 256, 0, c->stream>>>(p, v, count);
  HS_CUDA(cudaGetLastError());
  launch_count(c);
}

static void assemble(hs_matrix* m, const double* h_pts, size_t dim, double sf2,
                     double inv2l2, double sn2) {
  hs_ctx* c = m->ctx;
  HS_REQUIRE(sf2 > 0.0 && sn2 > 0.0, HS_ERR_CONFIG,
             "kernel variances must be positive");
  HS_REQUIRE(dim > 0, HS_ERR_CONFIG, "dimension must be positive");
  if (m->local_tiles() == 0) return;
  double* d_pts = nullptr;
  const size_t bytes = m->n * dim * sizeof(double);
  HS_CUDA(cudaMallocAsync(&d_pts, bytes, c->stream));
  HS_CUDA(cudaMemcpyAsync(d_pts, h_pts, bytes, cudaMemcpyHostToDevice,
                          c->stream));
  const int b = (int)m->b;
  // ~8K elements per CTA: 256 threads x 32 rows for b = 256
  const int rows_per_cta = std::max(1, std::min(b, 8192 / b));
  dim3 grid((unsigned)m->local_tiles(), (unsigned)ceil_div(b, rows_per_cta));
  const int threads = std::min(256, std::max(32, (b + 31) / 32 * 32));
  if (dim == 2)
    assemble_se_kernel<2><<<grid, threads, 0, c->stream>>>(
        m->d, m->tile_lo, m->d_owned, (int64_t)m->n, b, d_pts, (int)dim, sf2, inv2l2,
        sn2, rows_per_cta);
  else
    assemble_se_kernel<0><<<grid, threads, 0, c->stream>>>(
        m->d, m->tile_lo, m->d_owned, (int64_t)m->n, b, d_pts, (int)dim, sf2, inv2l2,
        sn2, rows_per_cta);
  HS_CUDA(cudaGetLastError());
  launch_count(c);
  HS_CUDA(cudaFreeAsync(d_pts, c->stream));
  HS_CUDA(cudaStreamSynchronize(c->stream));
  m->has_inv = false;
}

// ---- read-bandwidth probes (diagnostics) ----------------------------------

__global__ void __launch_bounds__(288, 1)
    probe_bulk_kernel(const double* __restrict__ src, int64_t slabs, double* sink) {
  constexpr int NS = 5, SLAB = 32768;
  extern __shared__ __align__(128) unsigned char psmem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(psmem + NS * SLAB);
  uint64_t* empty = full + NS;
  const int tid = threadIdx.x;
  const int64_t g0 = slabs * blockIdx.x / gridDim.x, g1 = slabs * (blockIdx.x + 1) / gridDim.x;
  if (tid == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 8);
    }
    fence_mbar_init();
  }
  __syncthreads();
  if (tid >= 256) {
    if (tid == 256)
      for (int64_t g = g0; g < g1; ++g) {
        const int64_t k = g - g0;
        const int st = (int)(k % NS);
        if (k >= NS) mbar_wait(&empty[st], (uint32_t)(((k / NS) - 1) & 1));
        mbar_arrive_expect_tx(&full[st], SLAB);
        bulk_g2s(psmem + st * SLAB, src + g * (SLAB / 8), SLAB, &full[st]);
      }
    return;
  }
  double acc = 0.0;
  for (int64_t g = g0; g < g1; ++g) {
    const int64_t k = g - g0;
    const int st = (int)(k % NS);
    mbar_wait(&full[st], (uint32_t)((k / NS) & 1));
    const double2* p = reinterpret_cast<const double2*>(psmem + st * SLAB);
#pragma unroll
    for (int m = 0; m < 8; ++m) {  // consumers read the slab like the SYMV
      const double2 v = p[tid + 256 * m];
      acc += v.x + v.y;
    }
    fence_proxy_async_smem();  // reads done before the refill
    __syncwarp();
    if ((tid & 31) == 0) mbar_arrive(&empty[st]);
  }
  if (acc == 123.456) *sink = acc;
}

__global__ void probe_ldg_kernel(const double2* __restrict__ src, int64_t n2, double* sink) {
  double acc = 0.0;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n2;
       k += (int64_t)gridDim.x * blockDim.x) {
    const double2 v = __ldcs(src + k);
    acc += v.x + v.y;
  }
  if (acc == 123.456) *sink = acc;
}

void* ctx_scratch(hs_ctx* c) {
  if (!c->scratch) {
    HS_CUDA(cudaMalloc(&c->scratch, 256));
    HS_CUDA(cudaMemset(c->scratch, 0, 256));
  }
  return c->scratch;
}

void ctx_workspace(hs_ctx* c, int slot, const size_t* sizes, int n, void** out) {
  auto up = [](size_t x) { return (x + 255) & ~(size_t)255; };
  size_t total = 0;
  for (int k = 0; k < n; ++k) total += up(sizes[k]);
  if (total > c->ws_bytes[slot]) {
    HS_CUDA(cudaDeviceSynchronize());  // the old buffer may be in use on any stream
    cudaFree(c->ws[slot]);
    c->ws[slot] = nullptr;
    c->ws_bytes[slot] = 0;
    HS_CUDA(cudaMalloc(&c->ws[slot], total));
    c->ws_bytes[slot] = total;
  }
  char* p = static_cast<char*>(c->ws[slot]);
  for (int k = 0; k < n; ++k) {
    out[k] = p;
    p += up(sizes[k]);
  }
}

double* ctx_vec(hs_ctx* c, int slot, size_t count) {
  if (c->vec_cap[slot] < count) {
    HS_CUDA(cudaStreamSynchronize(c->stream));
    cudaFree(c->vec[slot]);
    c->vec[slot] = nullptr;
    c->vec_cap[slot] = 0;
    HS_CUDA(cudaMalloc(&c->vec[slot], count * sizeof(double)));
    c->vec_cap[slot] = count;
  }
  return c->vec[slot];
}

// One communicator per context of a single-process group over distinct
// devices (ncclCommInitAll); rank r of the clique is ctxs[r].
void nccl_init_all(hs_ctx** ctxs, int world) {
  Nccl* n = load_nccl();
  std::vector<int> devs(world);
  for (int r = 0; r < world; ++r) devs[r] = ctxs[r]->device;
  std::vector<ncclComm_t> comms(world);
  nccl_check(n, n->CommInitAll(comms.data(), world, devs.data()), "ncclCommInitAll");
  for (int r = 0; r < world; ++r) {
    ctxs[r]->nccl = n;
    ctxs[r]->comm = comms[r];
  }
}

hs_matrix* cached_matrix(hs_ctx* c, int slot, size_t n, size_t b) {
  hs_matrix*& m = c->cache[slot];
  if (m && (m->n != n || m->b != b)) {
    hs_matrix_destroy(m);
    m = nullptr;
  }
  if (!m) {
    const hs_status s =
        slot >= 2 ? hs_matrix_create_cyclic(c, n, b, &m) : hs_matrix_create(c, n, b, &m);
    if (s != HS_OK) throw Failure{s, hs_last_error()};
  }
  m->has_inv = false;
  return m;
}

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

const char* hs_last_error(void) { return g_msg.c_str(); }
void hs_last_error_payload(int64_t* a, int64_t* b) {
  if (a) *a = g_pa;
  if (b) *b = g_pb;
}
const char* hs_error_kind_name(hs_status s) {
  switch (s) {
    case HS_OK: return "ok";
    case HS_ERR_CONFIG: return "config_error";
    case HS_ERR_NOT_SPD: return "not_spd";
    case HS_ERR_SINGULAR_BLOCK: return "singular_block";
    case HS_ERR_NUMERICAL: return "numerical_error";
    case HS_ERR_NOT_CONVERGED: return "not_converged";
    case HS_ERR_RESIDENCY: return "residency_error";
    case HS_ERR_FORMAT: return "format_error";
    case HS_ERR_VERSION_MISMATCH: return "version_mismatch";
    case HS_ERR_TRUNCATED_FILE: return "truncated_file";
    case HS_ERR_IO: return "io_error";
    case HS_ERR_CUDA: return "cuda_error";
  }
  return "unknown";
}

static void ctx_common_init(hs_ctx* c, int device, void* stream) {
  HS_CUDA(cudaSetDevice(device));
  c->device = device;
  if (stream) {
    c->stream = (cudaStream_t)stream;
  } else {
    HS_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    c->own_stream = true;
  }
  HS_CUDA(cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount,
                                 device));
  HS_CUDA(cudaMalloc(&c->d_scalars, sizeof(CgScalars)));
  // room for two CgScalars snapshots (the CG poll double-buffers them)
  HS_CUDA(cudaMallocHost(&c->h_pinned, std::max(64 * sizeof(double), 2 * sizeof(CgScalars))));
}

hs_status hs_device_alloc(hs_ctx* c, size_t bytes, void** out) {
  HS_API_BEGIN
  HS_REQUIRE(c && out, HS_ERR_CONFIG, "null pointer");
  HS_CUDA(cudaSetDevice(c->device));
  *out = nullptr;
  if (bytes) HS_CUDA(cudaMalloc(out, bytes));
  HS_API_END
}

void hs_device_free(hs_ctx* c, void* p) {
  if (!c || !p) return;
  cudaSetDevice(c->device);
  cudaStreamSynchronize(c->stream);
  cudaFree(p);
}

hs_status hs_memcpy(hs_ctx* c, void* dst, const void* src, size_t bytes) {
  HS_API_BEGIN
  HS_REQUIRE(c && (bytes == 0 || (dst && src)), HS_ERR_CONFIG, "null pointer");
  HS_CUDA(cudaSetDevice(c->device));
  if (bytes) HS_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, c->stream));
  HS_CUDA(cudaStreamSynchronize(c->stream));
  HS_API_END
}

hs_status hs_device_count(int* count) {
  HS_API_BEGIN
  HS_REQUIRE(count, HS_ERR_CONFIG, "null pointer");
  *count = 0;
  HS_CUDA(cudaGetDeviceCount(count));
  HS_API_END
}

hs_status hs_ctx_create(int device, void* stream, hs_ctx** out) {
  HS_API_BEGIN
  HS_REQUIRE(out, HS_ERR_CONFIG, "null output pointer");
  int count = 0;
  HS_CUDA(cudaGetDeviceCount(&count));
  HS_REQUIRE(device >= 0 && device < count, HS_ERR_CONFIG,
             "device index out of range");
  hs_ctx* c = new hs_ctx;
  try {
    ctx_common_init(c, device, stream);
  } catch (...) {
    delete c;
    throw;
  }
  *out = c;
  HS_API_END
}

hs_status hs_nccl_unique_id(void* id128) {
  HS_API_BEGIN
  Nccl* n = load_nccl();
  ncclUniqueId id;
  nccl_check(n, n->GetUniqueId(&id), "ncclGetUniqueId");
  static_assert(sizeof(ncclUniqueId) == 128, "nccl id size");
  std::memcpy(id128, &id, 128);
  HS_API_END
}

hs_status hs_ctx_create_nccl(int device, void* stream, int rank, int world,
                             const void* id128, hs_ctx** out) {
  HS_API_BEGIN
  HS_REQUIRE(out && id128, HS_ERR_CONFIG, "null pointer");
  HS_REQUIRE(world >= 1 && rank >= 0 && rank < world, HS_ERR_CONFIG,
             "bad rank/world");
  hs_ctx* c = new hs_ctx;
  try {
    ctx_common_init(c, device, stream);
    c->rank = rank;
    c->world = world;
    c->nccl = load_nccl();
    ncclUniqueId id;
    std::memcpy(&id, id128, 128);
    ncclComm_t comm;
    nccl_check(c->nccl, c->nccl->CommInitRank(&comm, world, id, rank),
               "ncclCommInitRank");
    c->comm = comm;
  } catch (...) {
    delete c;
    throw;
  }
  *out = c;
  HS_API_END
}

hs_status hs_ctx_create_custom_comm(int device, void* stream, int rank, int world,
                                    const hs_comm_ops* ops, hs_ctx** out) {
  HS_API_BEGIN
  HS_REQUIRE(out && ops && ops->allgather && ops->reduce_scatter && ops->broadcast &&
                 ops->allreduce_max_i64,
             HS_ERR_CONFIG, "null pointer / missing collective");
  HS_REQUIRE(world >= 1 && rank >= 0 && rank < world, HS_ERR_CONFIG, "bad rank/world");
  hs_ctx* c = new hs_ctx;
  try {
    ctx_common_init(c, device, stream);
    c->rank = rank;
    c->world = world;
    c->ops = *ops;
    c->custom = true;
  } catch (...) {
    delete c;
    throw;
  }
  *out = c;
  HS_API_END
}

hs_status hs_ctx_trim(hs_ctx* c) {
  HS_API_BEGIN
  HS_REQUIRE(c, HS_ERR_CONFIG, "null context");
  HS_CUDA(cudaSetDevice(c->device));
  HS_CUDA(cudaStreamSynchronize(c->stream));
  for (hs_matrix*& m : c->cache) {
    hs_matrix_destroy(m);
    m = nullptr;
  }
  cudaFree(c->cg_ws);
  c->cg_ws = nullptr;
  c->cg_ws_bytes = 0;
  delete c->oz_panel;
  c->oz_panel = nullptr;
  free_stager(c);
  for (int k = 0; k < 4; ++k) {
    cudaFree(c->vec[k]);
    c->vec[k] = nullptr;
    c->vec_cap[k] = 0;
    cudaFree(c->ws[k]);
    c->ws[k] = nullptr;
    c->ws_bytes[k] = 0;
  }
  HS_API_END
}

void hs_ctx_destroy(hs_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  cudaStreamSynchronize(c->stream);
  for (hs_matrix*& m : c->cache) {
    hs_matrix_destroy(m);
    m = nullptr;
  }
  if (c->comm) c->nccl->CommDestroy((ncclComm_t)c->comm);
  local_comm_release(c);
  for (cudaEvent_t e : c->prof_events) cudaEventDestroy(e);
  cudaFree(c->d_scalars);
  cudaFree(c->d_dpart);
  cudaFree(c->cg_ws);
  cudaFree(c->scratch);
  delete c->oz_panel;
  free_stager(c);
  for (double* v : c->vec) cudaFree(v);
  for (void* w : c->ws) cudaFree(w);
  cudaFreeHost(c->h_pinned);
  if (c->own_stream) cudaStreamDestroy(c->stream);
  delete c;
}

int hs_ctx_rank(const hs_ctx* c) { return c ? c->rank : -1; }
int hs_ctx_world(const hs_ctx* c) { return c ? c->world : 0; }
void* hs_ctx_stream(const hs_ctx* c) { return c ? (void*)c->stream : nullptr; }
uint64_t hs_ctx_kernel_launches(const hs_ctx* c) { return c ? c->launches : 0; }

hs_status hs_ctx_set_cholesky_gemm(hs_ctx* c, int slices) {
  HS_API_BEGIN
  HS_REQUIRE(c, HS_ERR_CONFIG, "null context");
  HS_REQUIRE(slices >= 0 && slices <= 8, HS_ERR_CONFIG,
             "Cholesky GEMM slices must be 0 (FP64 DMMA) or 1..8 (INT8 emulation)");
  c->chol_slices = slices;
  HS_API_END
}

size_t hs_ctx_ledger_size(const hs_ctx* c) { return c ? c->ledger.size() : 0; }
size_t hs_ctx_ledger_read(const hs_ctx* c, hs_ledger_entry* out, size_t cap) {
  if (!c || !out) return 0;
  const size_t k = std::min(cap, c->ledger.size());
  std::copy(c->ledger.begin(), c->ledger.begin() + k, out);
  return k;
}
void hs_ctx_ledger_clear(hs_ctx* c) {
  if (c) c->ledger.clear();
}

uint64_t hs_rng_at(uint64_t key, uint64_t counter) { return rng_at(key, counter); }
double hs_rng_uniform_pm1(uint64_t key, uint64_t counter) {
  return uniform_pm1(key, counter);
}

hs_status hs_generate_inputs(size_t n, size_t dim, uint64_t seed, double* out) {
  HS_API_BEGIN
  HS_REQUIRE(n > 0 && dim > 0, HS_ERR_CONFIG,
             "point count and dimension must be positive");
  gen_inputs(n, dim, seed, out);
  HS_API_END
}

double hs_median_pairwise_distance(const double* pts, size_t n, size_t dim) {
  return median_dist(pts, n, dim);
}

hs_status hs_generate_rhs(size_t n, size_t b, uint64_t seed, double* out) {
  HS_API_BEGIN
  HS_REQUIRE(n > 0 && b > 0, HS_ERR_CONFIG,
             "vector size and block size must be positive");
  const size_t pn = (size_t)ceil_div(n, b) * b;
  std::memset(out, 0, pn * sizeof(double));
  for (size_t i = 0; i < n; ++i) out[i] = uniform_pm1(seed ^ kRhsStream, i);
  HS_API_END
}

hs_status hs_partition_for_fraction(double f, size_t rows, size_t* split) {
  HS_API_BEGIN
  HS_REQUIRE(f >= 0.0 && f <= 1.0, HS_ERR_CONFIG,
             "split fraction must be in [0, 1], got " + std::to_string(f));
  HS_REQUIRE(rows > 0, HS_ERR_CONFIG,
             "partition requires at least one block row");
  *split = (size_t)floor(f * (double)rows + 0.5);
  HS_API_END
}

hs_status hs_cholesky_border(double f, size_t column, size_t rows,
                             size_t* beta) {
  HS_API_BEGIN
  HS_REQUIRE(f >= 0.0 && f <= 1.0, HS_ERR_CONFIG,
             "split fraction must be in [0, 1], got " + std::to_string(f));
  HS_REQUIRE(column < rows, HS_ERR_CONFIG, "cholesky_border column out of range");
  const size_t t = rows - 1 - column;
  const double budget = f * (double)(t * (t + 1) / 2);
  size_t out = rows;
  for (size_t be = column + 1; be <= rows; ++be) {
    const size_t k = be - column;
    const size_t below = (t * (t + 1) - (k - 1) * k) / 2;
    if ((double)below <= budget) {
      out = be;
      break;
    }
  }
  *beta = out;
  HS_API_END
}

hs_status hs_partition_rows(size_t rows, int world, size_t* bounds) {
  HS_API_BEGIN
  HS_REQUIRE(rows > 0 && world >= 1, HS_ERR_CONFIG, "bad partition request");
  auto b = row_bounds((int64_t)rows, world);
  for (int g = 0; g <= world; ++g) bounds[g] = (size_t)b[g];
  HS_API_END
}

hs_status hs_matrix_create(hs_ctx* c, size_t n, size_t b, hs_matrix** out) {
  HS_API_BEGIN
  HS_REQUIRE(c && out, HS_ERR_CONFIG, "null pointer");
  HS_REQUIRE(n > 0 && b > 0, HS_ERR_CONFIG,
             "matrix size and block size must be positive");
  HS_CUDA(cudaSetDevice(c->device));
  hs_matrix* m = new hs_matrix;
  m->ctx = c;
  m->n = n;
  m->b = b;
  m->N = (size_t)ceil_div(n, b);
  m->bounds = row_bounds((int64_t)m->N, c->world);
  if (c->world == 2 && c->row_fraction > 0.0 && c->row_fraction < 1.0 && m->N >= 2) {
    // the reference's executor split (partition.cpp:11-22): rank 0 plays B
    // (block rows [0, split)), rank 1 plays A ([split, N)); each rank keeps
    // at least one block row
    const int64_t split = (int64_t)floor(c->row_fraction * (double)m->N + 0.5);
    m->bounds[1] = std::min<int64_t>(std::max<int64_t>(split, 1), (int64_t)m->N - 1);
  }
  m->row_lo = (size_t)m->bounds[c->rank];
  m->row_hi = (size_t)m->bounds[c->rank + 1];
  m->tile_lo = tri((int64_t)m->row_lo, 0);
  m->tile_hi = tri((int64_t)m->row_hi, 0);
  // padded rank-chunk vector layout (identity for world == 1)
  int64_t lmax = 0;
  for (int g = 0; g < c->world; ++g)
    lmax = std::max<int64_t>(lmax, m->bounds[g + 1] - m->bounds[g]);
  m->slot_off = lmax * (int64_t)b;
  const int64_t stride = m->slot_off + (c->distributed() ? 2 * (int64_t)c->world : 0);
  m->vec_len = stride * c->world;
  std::vector<int64_t> off(m->N);
  for (int g = 0; g < c->world; ++g)
    for (int64_t i = m->bounds[g]; i < m->bounds[g + 1]; ++i)
      off[i] = (int64_t)g * stride + (i - m->bounds[g]) * (int64_t)b;
  try {
    const size_t bytes = m->local_tiles() * b * b * sizeof(double);
    if (bytes) HS_CUDA(cudaMalloc(&m->d, bytes));
    HS_CUDA(cudaMalloc(&m->d_row_off, m->N * sizeof(int64_t)));
    HS_CUDA(cudaMemcpy(m->d_row_off, off.data(), m->N * sizeof(int64_t),
                       cudaMemcpyHostToDevice));
    if (bytes) {
      HS_CUDA(cudaMemsetAsync(m->d, 0, bytes, c->stream));
      if (m->row_hi == m->N && m->N * b != n) {
        identity_pad_kernel<<<(unsigned)m->N, 256, 0, c->stream>>>(
            m->d, m->tile_lo, nullptr, (int64_t)n, (int)b, (int64_t)m->N);
        HS_CUDA(cudaGetLastError());
        launch_count(c);
      }
      HS_CUDA(cudaStreamSynchronize(c->stream));
    }
  } catch (...) {
    cudaFree(m->d);
    cudaFree(m->d_row_off);
    delete m;
    throw;
  }
  *out = m;
  HS_API_END
}

hs_status hs_matrix_create_cyclic(hs_ctx* c, size_t n, size_t b, hs_matrix** out) {
  HS_API_BEGIN
  HS_REQUIRE(c && out, HS_ERR_CONFIG, "null pointer");
  HS_REQUIRE(n > 0 && b > 0, HS_ERR_CONFIG,
             "matrix size and block size must be positive");
  HS_CUDA(cudaSetDevice(c->device));
  hs_matrix* m = new hs_matrix;
  m->ctx = c;
  m->n = n;
  m->b = b;
  m->N = (size_t)ceil_div(n, b);
  m->layout = 1;
  cyclic_grid(c->world, &m->P, &m->Q);
  const int64_t N = (int64_t)m->N, T = tri(N, 0);
  m->lpos.assign(T, -1);
  std::vector<int64_t> last_row_slot(N, -1);
  for (int64_t i = 0; i < N; ++i)
    for (int64_t j = 0; j <= i; ++j)
      if (cyclic_owner(i, j, m->P, m->Q) == c->rank) {
        m->lpos[tri(i, j)] = (int64_t)m->owned.size();
        if (i == N - 1) last_row_slot[j] = (int64_t)m->owned.size();
        m->owned.push_back(tri(i, j));
      }
  m->row_lo = 0;
  m->row_hi = m->N;
  m->tile_lo = 0;
  m->tile_hi = T;
  m->bounds = {0, (int64_t)m->N};
  m->vec_len = (int64_t)(m->N * b);
  m->slot_off = m->vec_len;
  try {
    const size_t bytes = m->local_tiles() * b * b * sizeof(double);
    if (bytes) HS_CUDA(cudaMalloc(&m->d, bytes));
    HS_CUDA(cudaMalloc(&m->d_owned, std::max<size_t>(1, m->owned.size()) * sizeof(int64_t)));
    HS_CUDA(cudaMalloc(&m->d_lpos, T * sizeof(int64_t)));
    HS_CUDA(cudaMemcpy(m->d_lpos, m->lpos.data(), T * sizeof(int64_t), cudaMemcpyHostToDevice));
    // vectors are full length on every rank: block row i at i * b (the SYMV
    // of a 1x1 grid, i.e. world 1, reads it)
    std::vector<int64_t> off(N);
    for (int64_t i = 0; i < N; ++i) off[i] = i * (int64_t)b;
    HS_CUDA(cudaMalloc(&m->d_row_off, N * sizeof(int64_t)));
    HS_CUDA(cudaMemcpy(m->d_row_off, off.data(), N * sizeof(int64_t), cudaMemcpyHostToDevice));
    if (!m->owned.empty())
      HS_CUDA(cudaMemcpy(m->d_owned, m->owned.data(), m->owned.size() * sizeof(int64_t),
                         cudaMemcpyHostToDevice));
    if (bytes) {
      HS_CUDA(cudaMemsetAsync(m->d, 0, bytes, c->stream));
      if (m->N * b != n) {
        int64_t* d_slot = nullptr;
        HS_CUDA(cudaMalloc(&d_slot, N * sizeof(int64_t)));
        HS_CUDA(cudaMemcpy(d_slot, last_row_slot.data(), N * sizeof(int64_t),
                           cudaMemcpyHostToDevice));
        identity_pad_kernel<<<(unsigned)N, 256, 0, c->stream>>>(m->d, 0, d_slot, (int64_t)n,
                                                                (int)b, N);
        HS_CUDA(cudaGetLastError());
        launch_count(c);
        HS_CUDA(cudaStreamSynchronize(c->stream));
        cudaFree(d_slot);
      }
      HS_CUDA(cudaStreamSynchronize(c->stream));
    }
  } catch (...) {
    cudaFree(m->d);
    cudaFree(m->d_owned);
    cudaFree(m->d_lpos);
    cudaFree(m->d_row_off);
    delete m;
    throw;
  }
  *out = m;
  HS_API_END
}

void hs_matrix_destroy(hs_matrix* m) {
  if (!m) return;
  cudaSetDevice(m->ctx->device);
  cudaStreamSynchronize(m->ctx->stream);
  if (m->plan) free_plan(m->plan);
  cudaFree(m->d_owned);
  cudaFree(m->d_lpos);
  cudaFree(m->d);
  cudaFree(m->dinv);
  cudaFree(m->d_row_off);
  delete m;
}

hs_status hs_matrix_info(const hs_matrix* m, size_t* n, size_t* b,
                         size_t* row_lo, size_t* row_hi) {
  HS_API_BEGIN
  HS_REQUIRE(m, HS_ERR_CONFIG, "null matrix");
  if (n) *n = m->n;
  if (b) *b = m->b;
  if (row_lo) *row_lo = m->row_lo;
  if (row_hi) *row_hi = m->row_hi;
  HS_API_END
}

static void cyclic_copy(hs_matrix* m, double* host, bool to_device) {
  // owned tiles, merged into runs that are contiguous on both sides
  const size_t bb = m->b * m->b;
  std::vector<CopySeg> segs;
  for (size_t k = 0; k < m->owned.size(); ++k) {
    double* h = host + (size_t)m->owned[k] * bb;
    double* d = m->d + k * bb;
    if (!segs.empty() && static_cast<char*>(segs.back().host) + segs.back().bytes == (char*)h &&
        static_cast<char*>(segs.back().dev) + segs.back().bytes == (char*)d)
      segs.back().bytes += bb * sizeof(double);
    else
      segs.push_back({d, h, bb * sizeof(double)});
  }
  host_copy(m->ctx, segs, to_device);
}

hs_status hs_matrix_upload(hs_matrix* m, const double* host) {
  HS_API_BEGIN
  HS_REQUIRE(m && host, HS_ERR_CONFIG, "null pointer");
  if (m->layout == 1) {
    cyclic_copy(m, const_cast<double*>(host), true);
    m->has_inv = false;
    return HS_OK;
  }
  const size_t bytes = m->local_tiles() * m->b * m->b * sizeof(double);
  host_copy(m->ctx, {{m->d, const_cast<double*>(host) + (size_t)m->tile_lo * m->b * m->b, bytes}},
            true);
  m->has_inv = false;
  HS_API_END
}

hs_status hs_matrix_download(const hs_matrix* m, double* host) {
  HS_API_BEGIN
  HS_REQUIRE(m && host, HS_ERR_CONFIG, "null pointer");
  if (m->layout == 1) {
    cyclic_copy(const_cast<hs_matrix*>(m), host, false);
    return HS_OK;
  }
  const size_t bytes = m->local_tiles() * m->b * m->b * sizeof(double);
  host_copy(m->ctx, {{m->d, host + (size_t)m->tile_lo * m->b * m->b, bytes}}, false);
  HS_API_END
}

hs_status hs_matrix_copy(hs_matrix* dst, const hs_matrix* src) {
  HS_API_BEGIN
  HS_REQUIRE(dst && src, HS_ERR_CONFIG, "null pointer");
  HS_REQUIRE(dst->ctx == src->ctx && dst->n == src->n && dst->b == src->b &&
                 dst->layout == src->layout,
             HS_ERR_CONFIG, "matrix shapes do not match");
  const size_t bytes = src->local_tiles() * src->b * src->b * sizeof(double);
  if (bytes)
    HS_CUDA(cudaMemcpyAsync(dst->d, src->d, bytes, cudaMemcpyDeviceToDevice,
                            src->ctx->stream));
  HS_CUDA(cudaStreamSynchronize(src->ctx->stream));
  dst->has_inv = false;
  HS_API_END
}

double* hs_matrix_device_data(hs_matrix* m) { return m ? m->d : nullptr; }

hs_status hs_assemble_se(hs_matrix* m, const double* points, size_t dim,
                         double sf2, double inv2l2, double sn2) {
  HS_API_BEGIN
  HS_REQUIRE(m && points, HS_ERR_CONFIG, "null pointer");
  HS_CUDA(cudaSetDevice(m->ctx->device));
  assemble(m, points, dim, sf2, inv2l2, sn2);
  HS_API_END
}

hs_status hs_generate_spd(hs_matrix* m, double sf2, double length_scale,
                          double sn2, size_t dim, uint64_t seed) {
  HS_API_BEGIN
  HS_REQUIRE(m, HS_ERR_CONFIG, "null matrix");
  HS_REQUIRE(sf2 > 0.0 && sn2 > 0.0, HS_ERR_CONFIG,
             "kernel variances must be positive");
  HS_REQUIRE(dim > 0, HS_ERR_CONFIG,
             "point count and dimension must be positive");
  HS_CUDA(cudaSetDevice(m->ctx->device));
  std::vector<double> pts(m->n * dim);
  gen_inputs(m->n, dim, seed, pts.data());
  const double ell =
      length_scale > 0.0 ? length_scale : median_dist(pts.data(), m->n, dim);
  assemble(m, pts.data(), dim, sf2, 1.0 / (2.0 * ell * ell), sn2);
  HS_API_END
}

hs_status hs_probe_hbm_read(hs_ctx* c, size_t bytes, int mode, int reps,
                            double* gbs) {
  HS_API_BEGIN
  HS_REQUIRE(c && gbs && bytes >= (1u << 20), HS_ERR_CONFIG, "bad probe arguments");
  HS_CUDA(cudaSetDevice(c->device));
  bytes &= ~size_t(32767);
  double* buf = nullptr;
  double* sink = nullptr;
  HS_CUDA(cudaMalloc(&buf, bytes));
  HS_CUDA(cudaMalloc(&sink, 8));
  cudaEvent_t e0, e1;
  HS_CUDA(cudaEventCreate(&e0));
  HS_CUDA(cudaEventCreate(&e1));
  HS_CUDA(cudaMemsetAsync(buf, 0, bytes, c->stream));
  const int smem = 5 * 32768 + 128;
  HS_CUDA(cudaFuncSetAttribute(probe_bulk_kernel,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  float best = 1e30f;
  for (int r = 0; r < std::max(reps, 1) + 1; ++r) {
    HS_CUDA(cudaEventRecord(e0, c->stream));
    if (mode == 0)
      probe_bulk_kernel<<<c->num_sms, 288, smem, c->stream>>>(buf, (int64_t)(bytes / 32768),
                                                              sink);
    else
      probe_ldg_kernel<<<c->num_sms * 8, 512, 0, c->stream>>>(
          reinterpret_cast<const double2*>(buf), (int64_t)(bytes / 16), sink);
    HS_CUDA(cudaGetLastError());
    HS_CUDA(cudaEventRecord(e1, c->stream));
    HS_CUDA(cudaEventSynchronize(e1));
    float ms = 0.f;
    HS_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    if (r > 0) best = std::min(best, ms);  // first run is a warm-up
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(buf);
  cudaFree(sink);
  *gbs = (double)bytes / (best * 1e-3) / 1e9;
  HS_API_END
}

void hs_prof_enable(hs_ctx* c, int every) {
  if (!c) return;
  c->prof = every > 0;
  c->prof_every = every > 0 ? every : 1;
  c->prof_counter = 0;
}

void hs_prof_symv(hs_ctx* c, uint64_t* launches, double* total_ms) {
  if (!c) return;
  cudaSetDevice(c->device);
  cudaStreamSynchronize(c->stream);
  for (size_t k = 0; k + 1 < c->prof_events.size(); k += 2) {
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, c->prof_events[k], c->prof_events[k + 1]) ==
        cudaSuccess) {
      c->prof_symv_ms += ms;
      c->prof_symv_launches += 1;
    }
    cudaEventDestroy(c->prof_events[k]);
    cudaEventDestroy(c->prof_events[k + 1]);
  }
  c->prof_events.clear();
  if (launches) *launches = c->prof_symv_launches;
  if (total_ms) *total_ms = c->prof_symv_ms;
}

void hs_prof_reset(hs_ctx* c) {
  if (!c) return;
  uint64_t l;
  double ms;
  hs_prof_symv(c, &l, &ms);
  c->prof_symv_launches = 0;
  c->prof_symv_ms = 0.0;
}

}  // extern "C"
