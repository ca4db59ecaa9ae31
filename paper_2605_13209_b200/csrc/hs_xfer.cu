// Host <-> device transfers of the host-buffer entry points.
//
// The reference API hands the solver std::vector storage: pageable memory.
// A plain cudaMemcpy from pageable memory goes through the driver's own
// bounce buffer at ~11 GB/s on a B200 host (measured, tools/h2d_probe.py),
// against ~55 GB/s from pinned memory. For pageable sources / destinations
// the copy is therefore staged: T host threads each own two pinned buffers
// and a stream; a thread copies its pieces host <-> pinned with memcpy while
// its other buffer's DMA is in flight. Pinned (page-locked or registered)
// buffers go straight to cudaMemcpyAsync.
#include <algorithm>
#include <cstring>
#include <thread>
#include <vector>

#include "hs_internal.h"

namespace hs {

struct HostStager {
  static constexpr size_t kBuf = 8u << 20;  // bytes per pinned buffer
  int device = 0;
  int threads = 0;
  std::vector<cudaStream_t> streams;   // [threads]
  std::vector<void*> bufs;             // [threads][2]
  std::vector<cudaEvent_t> events;     // [threads][2]
  ~HostStager() {
    cudaSetDevice(device);
    for (cudaStream_t s : streams) cudaStreamSynchronize(s);
    for (cudaEvent_t e : events) cudaEventDestroy(e);
    for (void* p : bufs) cudaFreeHost(p);
    for (cudaStream_t s : streams) cudaStreamDestroy(s);
  }
};

static HostStager& stager(hs_ctx* c) {
  if (!c->stager) {
    HostStager* st = new HostStager;
    st->device = c->device;
    st->threads = (int)std::max(2u, std::min(8u, std::thread::hardware_concurrency() / 2));
    try {
      for (int t = 0; t < st->threads; ++t) {
        cudaStream_t s;
        HS_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
        st->streams.push_back(s);
        for (int k = 0; k < 2; ++k) {
          void* p = nullptr;
          HS_CUDA(cudaHostAlloc(&p, HostStager::kBuf, cudaHostAllocDefault));
          st->bufs.push_back(p);
          cudaEvent_t e;
          HS_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
          st->events.push_back(e);
        }
      }
    } catch (...) {
      delete st;
      throw;
    }
    c->stager = st;
  }
  return *c->stager;
}

void free_stager(hs_ctx* c) {
  delete c->stager;
  c->stager = nullptr;
}

static bool is_pinned(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

void host_copy(hs_ctx* c, const std::vector<CopySeg>& segs, bool h2d) {
  size_t total = 0;
  for (const CopySeg& s : segs) total += s.bytes;
  if (!total) return;
  const cudaMemcpyKind kind = h2d ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToHost;
  if (is_pinned(segs.front().host) || total < (4u << 20)) {
    for (const CopySeg& s : segs)
      HS_CUDA(cudaMemcpyAsync(h2d ? s.dev : s.host, h2d ? s.host : s.dev, s.bytes, kind,
                              c->stream));
    HS_CUDA(cudaStreamSynchronize(c->stream));
    return;
  }
  HostStager& st = stager(c);
  // pieces of at most one buffer, in segment order
  struct Piece {
    char* dev;
    char* host;
    size_t bytes;
  };
  std::vector<Piece> pieces;
  for (const CopySeg& s : segs)
    for (size_t o = 0; o < s.bytes; o += HostStager::kBuf)
      pieces.push_back({static_cast<char*>(s.dev) + o, static_cast<char*>(s.host) + o,
                        std::min(HostStager::kBuf, s.bytes - o)});
  // device work queued on the context stream (e.g. a factorization) must be
  // finished before a download reads the matrix
  HS_CUDA(cudaStreamSynchronize(c->stream));
  const int T = std::min<int>(st.threads, (int)pieces.size());
  std::vector<cudaError_t> err(T, cudaSuccess);
  auto work = [&](int t) {
    cudaError_t e = cudaSetDevice(st.device);
    cudaStream_t s = st.streams[t];
    void* buf[2] = {st.bufs[2 * t], st.bufs[2 * t + 1]};
    cudaEvent_t ev[2] = {st.events[2 * t], st.events[2 * t + 1]};
    int k = 0;
    const Piece* pend = nullptr;  // download: piece whose DMA is in flight
    int pend_slot = 0;
    for (size_t i = t; i < pieces.size() && e == cudaSuccess; i += T, ++k) {
      const Piece& p = pieces[i];
      const int slot = k & 1;
      if (h2d) {
        // the buffer's previous DMA must be done before it is refilled
        if (k >= 2) e = cudaEventSynchronize(ev[slot]);
        if (e != cudaSuccess) break;
        std::memcpy(buf[slot], p.host, p.bytes);
        e = cudaMemcpyAsync(p.dev, buf[slot], p.bytes, cudaMemcpyHostToDevice, s);
        if (e == cudaSuccess) e = cudaEventRecord(ev[slot], s);
      } else {
        e = cudaMemcpyAsync(buf[slot], p.dev, p.bytes, cudaMemcpyDeviceToHost, s);
        if (e == cudaSuccess) e = cudaEventRecord(ev[slot], s);
        if (e == cudaSuccess && pend) {
          e = cudaEventSynchronize(ev[pend_slot]);
          if (e == cudaSuccess) std::memcpy(pend->host, buf[pend_slot], pend->bytes);
        }
        pend = &p;
        pend_slot = slot;
      }
    }
    if (e == cudaSuccess && pend) {
      e = cudaEventSynchronize(ev[pend_slot]);
      if (e == cudaSuccess) std::memcpy(pend->host, buf[pend_slot], pend->bytes);
    }
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    err[t] = e;
  };
  std::vector<std::thread> pool;
  for (int t = 1; t < T; ++t) pool.emplace_back(work, t);
  work(0);
  for (std::thread& th : pool) th.join();
  for (cudaError_t e : err)
    if (e != cudaSuccess)
      throw Failure{HS_ERR_CUDA, std::string("staged host copy: ") + cudaGetErrorString(e)};
}

}  // namespace hs
