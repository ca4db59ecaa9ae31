// Single-process multi-GPU groups (the reference's `Runtime` with its two
// executors, executor.hpp:128-221, generalised to G devices driven from one
// process): one hs_ctx per rank, one host thread per rank while a solve
// runs, and the collectives of the distributed CG / Cholesky either over
// NCCL (ncclCommInitAll, distinct devices) or over the in-process transport
// below.
//
// In-process transport ("local"): every collective is an issue-time
// rendezvous of the rank threads followed by device copies ordered with CUDA
// events, so nothing blocks the host on the GPU and nothing synchronizes a
// stream -- the same asynchronous stream semantics as NCCL, which the
// blocking host-callback transport of hs_ctx_create_custom_comm hides. Per
// collective:
//   1. each rank records `ready` on the issuing stream (its send buffer is
//      produced) and publishes (send, recv, ready, done);
//   2. barrier A;
//   3. each rank enqueues, on its own stream, waits on the peers' `ready`
//      and the copies it needs from their send buffers into its receive
//      buffer (or staging + a fixed rank-order reduction kernel), then
//      records `done`;
//   4. barrier B; each rank's stream waits on every peer's `done`, so no
//      rank overwrites a buffer a peer still reads.
// Events and slots are double buffered by collective parity: a rank can run
// at most one collective ahead of the slowest (barrier A). Ranks may share a
// device, which is how the multi-rank code paths are tested on one GPU with
// real stream overlap (Cholesky lookahead streams included).
#include <algorithm>
#include <chrono>
#include <condition_variable>
#include <cstring>
#include <mutex>
#include <thread>
#include <vector>

#include "hs_internal.h"

namespace hs {

struct LocalShared {
  int world = 1;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t gen = 0;
  bool aborted = false;
  struct Slot {
    const void* send = nullptr;
    void* recv = nullptr;
    cudaEvent_t ready = nullptr, done = nullptr;
  };
  std::vector<Slot> slots[2];  // by collective parity

  void wait() {
    std::unique_lock<std::mutex> lk(mu);
    if (aborted) throw Failure{HS_ERR_CUDA, "group collective aborted: another rank failed"};
    const uint64_t g = gen;
    if (++arrived == world) {
      arrived = 0;
      ++gen;
      cv.notify_all();
      return;
    }
    cv.wait(lk, [&] { return gen != g || aborted; });
    if (gen == g) throw Failure{HS_ERR_CUDA, "group collective aborted: another rank failed"};
  }
  void abort() {
    std::lock_guard<std::mutex> lk(mu);
    aborted = true;
    cv.notify_all();
  }
  void reset() {
    std::lock_guard<std::mutex> lk(mu);
    aborted = false;
    arrived = 0;
  }
};

struct LocalComm {
  LocalShared* sh = nullptr;
  int rank = 0;
  uint64_t seq = 0;
  cudaEvent_t ready[2] = {nullptr, nullptr}, done[2] = {nullptr, nullptr};
  void* stage = nullptr;  // reduction staging (world * count elements)
  size_t stage_bytes = 0;
  void* snap = nullptr;   // all-reduce send snapshot
  size_t snap_bytes = 0;
};

static void* grow(void*& p, size_t& cap, size_t bytes) {
  if (cap < bytes) {
    cudaFree(p);  // implicit device sync: rare (buffers only grow)
    p = nullptr;
    cap = 0;
    HS_CUDA(cudaMalloc(&p, bytes));
    cap = bytes;
  }
  return p;
}

template <class Pre, class Body>
static void collective(hs_ctx* c, cudaStream_t s, const void* send, void* recv, Pre pre,
                       Body body) {
  LocalComm* L = c->local;
  LocalShared* S = L->sh;
  const int par = (int)(L->seq++ & 1);
  pre();
  HS_CUDA(cudaEventRecord(L->ready[par], s));
  S->slots[par][L->rank] = LocalShared::Slot{send, recv, L->ready[par], L->done[par]};
  S->wait();  // A: every rank's send buffer is published
  body(S->slots[par]);
  HS_CUDA(cudaEventRecord(L->done[par], s));
  S->wait();  // B: every rank has enqueued its reads
  for (int g = 0; g < S->world; ++g)
    if (g != L->rank) HS_CUDA(cudaStreamWaitEvent(s, S->slots[par][g].done, 0));
}

__global__ void rank_sum_f64(const double* stage, double* out, int64_t count, int world) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < count;
       k += (int64_t)gridDim.x * blockDim.x) {
    double v = stage[k];
    for (int g = 1; g < world; ++g) v += stage[g * count + k];  // rank order
    out[k] = v;
  }
}

__global__ void rank_max_i64(const int64_t* stage, int64_t* out, int64_t count, int world) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < count;
       k += (int64_t)gridDim.x * blockDim.x) {
    int64_t v = stage[k];
    for (int g = 1; g < world; ++g) v = max(v, stage[g * count + k]);
    out[k] = v;
  }
}

static unsigned grid_for(int64_t count) {
  return (unsigned)std::min<int64_t>(4 * 148, std::max<int64_t>(1, (count + 255) / 256));
}

void local_allgather(hs_ctx* c, const double* send, double* recv, size_t count,
                     cudaStream_t s) {
  const int me = c->local->rank;
  const size_t bytes = count * sizeof(double);
  collective(c, s, send, recv, [] {}, [&](const std::vector<LocalShared::Slot>& sl) {
    for (int g = 0; g < (int)sl.size(); ++g) {
      double* dst = recv + (size_t)g * count;
      if (g == me) {
        if (send != dst && bytes)
          HS_CUDA(cudaMemcpyAsync(dst, send, bytes, cudaMemcpyDefault, s));
        continue;
      }
      HS_CUDA(cudaStreamWaitEvent(s, sl[g].ready, 0));
      if (bytes) HS_CUDA(cudaMemcpyAsync(dst, sl[g].send, bytes, cudaMemcpyDefault, s));
    }
  });
}

void local_reduce_scatter(hs_ctx* c, const double* send, double* recv, size_t count,
                          cudaStream_t s) {
  LocalComm* L = c->local;
  const int me = L->rank, world = L->sh->world;
  const size_t bytes = count * sizeof(double);
  double* stage = static_cast<double*>(grow(L->stage, L->stage_bytes, bytes * world));
  collective(c, s, send, recv, [] {}, [&](const std::vector<LocalShared::Slot>& sl) {
    for (int g = 0; g < world; ++g) {
      if (g != me) HS_CUDA(cudaStreamWaitEvent(s, sl[g].ready, 0));
      const double* src = static_cast<const double*>(sl[g].send) + (size_t)me * count;
      if (bytes)
        HS_CUDA(cudaMemcpyAsync(stage + (size_t)g * count, src, bytes, cudaMemcpyDefault, s));
    }
    if (count) {
      rank_sum_f64<<<grid_for((int64_t)count), 256, 0, s>>>(stage, recv, (int64_t)count,
                                                             world);
      HS_CUDA(cudaGetLastError());
      launch_count(c);
    }
  });
}

void local_bcast(hs_ctx* c, const double* send, double* recv, size_t count, int root,
                 cudaStream_t s) {
  const int me = c->local->rank;
  const size_t bytes = count * sizeof(double);
  collective(c, s, me == root ? send : nullptr, recv, [] {},
             [&](const std::vector<LocalShared::Slot>& sl) {
               if (!bytes) return;
               if (me == root) {
                 if (send != recv)
                   HS_CUDA(cudaMemcpyAsync(recv, send, bytes, cudaMemcpyDefault, s));
                 return;
               }
               HS_CUDA(cudaStreamWaitEvent(s, sl[root].ready, 0));
               HS_CUDA(cudaMemcpyAsync(recv, sl[root].send, bytes, cudaMemcpyDefault, s));
             });
}

void local_allreduce_max_i64(hs_ctx* c, int64_t* buf, size_t count, cudaStream_t s) {
  LocalComm* L = c->local;
  const int world = L->sh->world;
  const size_t bytes = count * sizeof(int64_t);
  int64_t* snap = static_cast<int64_t*>(grow(L->snap, L->snap_bytes, std::max<size_t>(bytes, 8)));
  int64_t* stage = static_cast<int64_t*>(grow(L->stage, L->stage_bytes, bytes * world));
  collective(
      c, s, snap, buf,
      [&] {  // peers read a snapshot: `buf` itself is overwritten below
        if (bytes) HS_CUDA(cudaMemcpyAsync(snap, buf, bytes, cudaMemcpyDeviceToDevice, s));
      },
      [&](const std::vector<LocalShared::Slot>& sl) {
        for (int g = 0; g < world; ++g) {
          if (g != L->rank) HS_CUDA(cudaStreamWaitEvent(s, sl[g].ready, 0));
          if (bytes)
            HS_CUDA(cudaMemcpyAsync(stage + (size_t)g * count, sl[g].send, bytes,
                                    cudaMemcpyDefault, s));
        }
        if (count) {
          rank_max_i64<<<grid_for((int64_t)count), 256, 0, s>>>(stage, buf, (int64_t)count,
                                                                 world);
          HS_CUDA(cudaGetLastError());
          launch_count(c);
        }
      });
}

void local_comm_release(hs_ctx* c) {
  LocalComm* L = c->local;
  if (!L) return;
  for (int k = 0; k < 2; ++k) {
    if (L->ready[k]) cudaEventDestroy(L->ready[k]);
    if (L->done[k]) cudaEventDestroy(L->done[k]);
  }
  cudaFree(L->stage);
  cudaFree(L->snap);
  delete L;
  c->local = nullptr;
}

}  // namespace hs

using namespace hs;

struct hs_group {
  int world = 1;
  int transport = 0;  // resolved: 0 none (world 1), 1 NCCL, 2 in-process
  std::vector<hs_ctx*> ctx;
  LocalShared* shared = nullptr;
  hs_ctx* solo = nullptr;  // plain context on ctx[0]'s device (unsupported shapes)
};

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

namespace {

struct RankResult {
  hs_status status = HS_OK;
  std::string msg;
  int64_t a = -1, b = -1;
};

// Runs fn(rank, ctx) on one host thread per rank; the first failing rank's
// error (in rank order) becomes the caller's. A rank that fails releases the
// others from the in-process transport's barriers.
template <class Fn>
void run_ranks(hs_group* g, Fn fn) {
  std::vector<RankResult> res(g->world);
  auto body = [&](int r) {
    cudaSetDevice(g->ctx[r]->device);
    clear_error();
    hs_status s = HS_OK;
    try {
      s = fn(r, g->ctx[r]);
    } catch (const Failure& f) {
      set_error(f.status, f.msg, f.a, f.b);
      s = f.status;
    } catch (const std::exception& e) {
      set_error(HS_ERR_CUDA, e.what());
      s = HS_ERR_CUDA;
    }
    if (s != HS_OK) {
      res[r].status = s;
      res[r].msg = hs_last_error();
      hs_last_error_payload(&res[r].a, &res[r].b);
      if (g->shared) g->shared->abort();
    }
  };
  if (g->world == 1) {
    body(0);
  } else {
    std::vector<std::thread> th;
    for (int r = 0; r < g->world; ++r) th.emplace_back(body, r);
    for (auto& t : th) t.join();
  }
  if (g->shared) g->shared->reset();
  // an agreed error (NotSpd / Numerical on every rank) beats a rank that was
  // only released from a barrier by another's failure
  const RankResult* pick = nullptr;
  for (const RankResult& r : res)
    if (r.status != HS_OK && r.msg.find("aborted: another rank failed") == std::string::npos) {
      pick = &r;
      break;
    }
  for (const RankResult& r : res)
    if (!pick && r.status != HS_OK) pick = &r;
  if (pick) throw Failure{pick->status, pick->msg, pick->a, pick->b};
}

// a shape the distributed paths do not serve runs on one GPU
bool dist_cg_ok(size_t b) { return b == 64 || b == 128 || b == 256 || b == 512; }
bool dist_chol_ok(size_t b) { return b % 128 == 0; }

hs_ctx* solo_ctx(hs_group* g) {
  if (!g->solo) {
    const hs_status s = hs_ctx_create(g->ctx[0]->device, nullptr, &g->solo);
    if (s != HS_OK) throw Failure{s, hs_last_error()};
  }
  return g->solo;
}

void clear_peer_ledgers(hs_group* g) {
  for (int r = 1; r < g->world; ++r) g->ctx[r]->ledger.clear();
}

}  // namespace

extern "C" {

hs_status hs_group_create(int world, const int* devices, int transport, hs_group** out) {
  HS_API_BEGIN
  HS_REQUIRE(out && world >= 1, HS_ERR_CONFIG, "bad group request");
  HS_REQUIRE(transport >= 0 && transport <= 2, HS_ERR_CONFIG,
             "transport must be 0 (auto), 1 (NCCL) or 2 (in-process)");
  int count = 0;
  HS_CUDA(cudaGetDeviceCount(&count));
  std::vector<int> dev(world);
  for (int r = 0; r < world; ++r) {
    dev[r] = devices ? devices[r] : r % std::max(count, 1);
    HS_REQUIRE(dev[r] >= 0 && dev[r] < count, HS_ERR_CONFIG, "device index out of range");
  }
  bool distinct = true;
  for (int r = 0; r < world; ++r)
    for (int q = 0; q < r; ++q) distinct &= dev[r] != dev[q];
  int t = world == 1 ? 0 : transport == 0 ? (distinct ? 1 : 2) : transport;
  HS_REQUIRE(!(t == 1 && !distinct), HS_ERR_CONFIG,
             "NCCL needs a distinct device per rank (use the in-process transport)");
  hs_group* g = new hs_group;
  g->world = world;
  g->transport = t;
  try {
    for (int r = 0; r < world; ++r) {
      hs_ctx* c = nullptr;
      const hs_status s = hs_ctx_create(dev[r], nullptr, &c);
      if (s != HS_OK) throw Failure{s, hs_last_error()};
      c->rank = r;
      c->world = world;
      g->ctx.push_back(c);
    }
    if (t == 1) {
      nccl_init_all(g->ctx.data(), world);
    } else if (t == 2) {
      g->shared = new LocalShared;
      g->shared->world = world;
      g->shared->slots[0].resize(world);
      g->shared->slots[1].resize(world);
      for (int r = 0; r < world; ++r) {
        hs_ctx* c = g->ctx[r];
        HS_CUDA(cudaSetDevice(c->device));
        LocalComm* L = new LocalComm;
        L->sh = g->shared;
        L->rank = r;
        c->local = L;
        for (int k = 0; k < 2; ++k) {
          HS_CUDA(cudaEventCreateWithFlags(&L->ready[k], cudaEventDisableTiming));
          HS_CUDA(cudaEventCreateWithFlags(&L->done[k], cudaEventDisableTiming));
        }
        // direct NVLink copies between distinct devices
        for (int q = 0; q < world; ++q) {
          int can = 0;
          if (dev[q] != c->device &&
              cudaDeviceCanAccessPeer(&can, c->device, dev[q]) == cudaSuccess && can) {
            const cudaError_t e = cudaDeviceEnablePeerAccess(dev[q], 0);
            if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
          }
        }
      }
    }
  } catch (...) {
    for (hs_ctx* c : g->ctx) hs_ctx_destroy(c);
    delete g->shared;
    delete g;
    throw;
  }
  *out = g;
  HS_API_END
}

void hs_group_destroy(hs_group* g) {
  if (!g) return;
  for (hs_ctx* c : g->ctx) hs_ctx_destroy(c);
  if (g->solo) hs_ctx_destroy(g->solo);
  delete g->shared;
  delete g;
}

int hs_group_world(const hs_group* g) { return g ? g->world : 0; }
int hs_group_transport(const hs_group* g) { return g ? g->transport : -1; }
hs_ctx* hs_group_ctx(hs_group* g, int rank) {
  return g && rank >= 0 && rank < g->world ? g->ctx[rank] : nullptr;
}

hs_status hs_group_set_row_fraction(hs_group* g, double fraction) {
  HS_API_BEGIN
  HS_REQUIRE(g, HS_ERR_CONFIG, "null group");
  HS_REQUIRE(fraction >= 0.0 && fraction <= 1.0, HS_ERR_CONFIG,
             "split fraction must be in [0, 1], got " + std::to_string(fraction));
  for (hs_ctx* c : g->ctx) {
    if (c->row_fraction != fraction) {
      // cached row-sharded matrices were partitioned for the old split
      cudaSetDevice(c->device);
      cudaStreamSynchronize(c->stream);
      for (int k = 0; k < 2; ++k) {
        hs_matrix_destroy(c->cache[k]);
        c->cache[k] = nullptr;
      }
    }
    c->row_fraction = fraction;
  }
  HS_API_END
}

hs_status hs_group_set_cholesky_gemm(hs_group* g, int slices) {
  HS_API_BEGIN
  HS_REQUIRE(g, HS_ERR_CONFIG, "null group");
  for (hs_ctx* c : g->ctx) {
    const hs_status s = hs_ctx_set_cholesky_gemm(c, slices);
    if (s != HS_OK) throw Failure{s, hs_last_error()};
  }
  if (g->solo) hs_ctx_set_cholesky_gemm(g->solo, slices);
  HS_API_END
}

hs_status hs_group_run(hs_group* g, int (*fn)(int rank, hs_ctx* ctx, void* arg), void* arg) {
  HS_API_BEGIN
  HS_REQUIRE(g && fn, HS_ERR_CONFIG, "null pointer");
  run_ranks(g, [&](int r, hs_ctx* c) { return (hs_status)fn(r, c, arg); });
  HS_API_END
}

hs_status hs_group_solve_cg_host(hs_group* g, size_t n, size_t b, const double* a,
                                 const double* rhs, const hs_cg_params* p, double* x,
                                 hs_cg_stats* st, double* trace) {
  HS_API_BEGIN
  HS_REQUIRE(g && a && rhs && p && x && st, HS_ERR_CONFIG, "null pointer");
  if (g->world > 1 && !dist_cg_ok(b)) {
    const hs_status s = hs_solve_cg_host(solo_ctx(g), n, b, a, rhs, p, x, st, trace);
    if (s != HS_OK) throw Failure{s, hs_last_error()};
    return HS_OK;
  }
  std::vector<hs_cg_stats> sts(g->world);
  const size_t pn = (size_t)ceil_div(n, b) * b;
  run_ranks(g, [&](int r, hs_ctx* c) {
    std::vector<double> xs(r == 0 ? 0 : pn);
    return hs_solve_cg_host(c, n, b, a, rhs, p, r == 0 ? x : xs.data(), &sts[r],
                            r == 0 ? trace : nullptr);
  });
  *st = sts[0];
  for (const hs_cg_stats& s : sts) {  // the job's times are the slowest rank's
    st->wall_ms = std::max(st->wall_ms, s.wall_ms);
    st->transfer_ms = std::max(st->transfer_ms, s.transfer_ms);
  }
  st->compute_ms = st->wall_ms - st->transfer_ms;
  clear_peer_ledgers(g);
  HS_API_END
}

// factorize / solve_spd over the group: 2D block-cyclic tiles, each rank
// uploads / downloads only its own tiles of the caller's packed array
hs_status hs_group_factorize_host(hs_group* g, size_t n, size_t b, double* a,
                                  hs_chol_stats* st) {
  HS_API_BEGIN
  HS_REQUIRE(g && a, HS_ERR_CONFIG, "null pointer");
  if (g->world > 1 && !dist_chol_ok(b)) {
    const hs_status s = hs_factorize_host(solo_ctx(g), n, b, a, st);
    if (s != HS_OK) throw Failure{s, hs_last_error()};
    return HS_OK;
  }
  std::vector<hs_chol_stats> sts(g->world);
  run_ranks(g, [&](int r, hs_ctx* c) {
    if (g->world == 1) return hs_factorize_host(c, n, b, a, &sts[r]);
    hs_matrix* m = cached_matrix(c, 2, n, b);
    const auto t0 = std::chrono::steady_clock::now();
    hs_status s = hs_matrix_upload(m, a);
    if (s != HS_OK) return s;
    const auto t1 = std::chrono::steady_clock::now();
    s = hs_potrf(c, m, nullptr);
    if (s != HS_OK) return s;
    const auto t2 = std::chrono::steady_clock::now();
    s = hs_matrix_download(m, a);
    const auto t3 = std::chrono::steady_clock::now();
    auto ms = [](auto u, auto v) { return std::chrono::duration<double, std::milli>(v - u).count(); };
    sts[r].compute_ms = ms(t1, t2);
    sts[r].transfer_ms = ms(t0, t1) + ms(t2, t3);
    sts[r].factor_ms = sts[r].wall_ms = ms(t0, t3);
    return s;
  });
  if (st) {
    *st = sts[0];
    for (const hs_chol_stats& s : sts) {
      st->wall_ms = std::max(st->wall_ms, s.wall_ms);
      st->factor_ms = std::max(st->factor_ms, s.factor_ms);
      st->compute_ms = std::max(st->compute_ms, s.compute_ms);
      st->transfer_ms = std::max(st->transfer_ms, s.transfer_ms);
    }
  }
  clear_peer_ledgers(g);
  HS_API_END
}

hs_status hs_group_solve_spd_host(hs_group* g, size_t n, size_t b, double* a,
                                  const double* rhs, double* x, hs_chol_stats* st) {
  HS_API_BEGIN
  HS_REQUIRE(g && a && rhs && x, HS_ERR_CONFIG, "null pointer");
  if (g->world > 1 && !dist_chol_ok(b)) {
    const hs_status s = hs_solve_spd_host(solo_ctx(g), n, b, a, rhs, x, st);
    if (s != HS_OK) throw Failure{s, hs_last_error()};
    return HS_OK;
  }
  std::vector<hs_chol_stats> sts(g->world);
  const size_t pn = (size_t)ceil_div(n, b) * b;
  run_ranks(g, [&](int r, hs_ctx* c) {
    if (g->world == 1) return hs_solve_spd_host(c, n, b, a, rhs, x, &sts[r]);
    hs_matrix* m = cached_matrix(c, 2, n, b);
    hs_matrix* orig = cached_matrix(c, 3, n, b);
    double* d_rhs = ctx_vec(c, 0, pn);
    double* d_x = ctx_vec(c, 1, pn);
    const auto t0 = std::chrono::steady_clock::now();
    hs_status s = hs_matrix_upload(m, a);
    if (s != HS_OK) return s;
    HS_CUDA(cudaMemcpyAsync(d_rhs, rhs, pn * sizeof(double), cudaMemcpyHostToDevice,
                            c->stream));
    s = hs_matrix_copy(orig, m);
    if (s != HS_OK) return s;
    const auto t1 = std::chrono::steady_clock::now();
    s = hs_solve_spd(c, m, d_rhs, d_x, orig, &sts[r]);
    if (s != HS_OK) return s;
    const auto t2 = std::chrono::steady_clock::now();
    if (r == 0)
      HS_CUDA(cudaMemcpyAsync(x, d_x, pn * sizeof(double), cudaMemcpyDeviceToHost,
                              c->stream));
    s = hs_matrix_download(m, a);
    HS_CUDA(cudaStreamSynchronize(c->stream));
    const auto t3 = std::chrono::steady_clock::now();
    auto ms = [](auto u, auto v) { return std::chrono::duration<double, std::milli>(v - u).count(); };
    sts[r].transfer_ms = ms(t0, t1) + ms(t2, t3);
    sts[r].wall_ms = ms(t0, t3);
    (void)t1;
    return s;
  });
  if (st) {
    *st = sts[0];
    for (const hs_chol_stats& s : sts) {
      st->wall_ms = std::max(st->wall_ms, s.wall_ms);
      st->factor_ms = std::max(st->factor_ms, s.factor_ms);
      st->solve_ms = std::max(st->solve_ms, s.solve_ms);
      st->transfer_ms = std::max(st->transfer_ms, s.transfer_ms);
    }
    st->compute_ms = st->wall_ms - st->transfer_ms;
  }
  clear_peer_ledgers(g);
  HS_API_END
}

}  // extern "C"
