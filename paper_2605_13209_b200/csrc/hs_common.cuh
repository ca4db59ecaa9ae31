// Shared device + host helpers for the B200 SPD-solve library
// (libhsolve_cuda.so). sm_100a only.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <string>
#include <utility>

#include "hs_cuda.h"

namespace hs {

// ---------------------------------------------------------------------------
// Error plumbing: every ABI entry converts failures into an HS_* status and a
// thread-local message (hs_last_error). Nothing throws across the ABI.

struct Failure {
  int status;
  std::string msg;
  int64_t a = -1, b = -1;  // payload (not_spd: block row / pivot, ...)
};

void set_error(int status, const std::string& msg, int64_t a = -1,
               int64_t b = -1);
void clear_error();

#define HS_CUDA(call)                                                        \
  do {                                                                       \
    cudaError_t e_ = (call);                                                 \
    if (e_ != cudaSuccess)                                                   \
      throw ::hs::Failure{HS_ERR_CUDA, std::string(#call) + ": " +           \
                                           cudaGetErrorString(e_)};          \
  } while (0)

#define HS_REQUIRE(cond, status, msg)                                        \
  do {                                                                       \
    if (!(cond)) throw ::hs::Failure{(status), (msg)};                       \
  } while (0)

// ---------------------------------------------------------------------------
// Packed lower-triangular tile indexing (reference blocked_matrix.cpp:8-15):
// tile (i, j), j <= i, lives at tri(i, j) * b * b; element (r, c) at r*b + c.

__host__ __device__ __forceinline__ int64_t tri(int64_t i, int64_t j) {
  return i * (i + 1) / 2 + j;
}

// Inverse of tri(i, 0): the block row that holds packed tile index t.
__host__ __device__ __forceinline__ int64_t tile_row(int64_t t) {
  int64_t i = (int64_t)((sqrt(8.0 * (double)t + 1.0) - 1.0) * 0.5);
  while (tri(i + 1, 0) <= t) ++i;
  while (tri(i, 0) > t) --i;
  return i;
}

// ---------------------------------------------------------------------------
// Double-double (Knuth TwoSum) — same operations as reference dd.hpp:18-40,
// with contraction explicitly disabled (__dadd_rn) so nvcc cannot fuse.

struct Dd {
  double hi, lo;
};

__host__ __device__ __forceinline__ Dd dd_two_sum(double a, double b) {
#ifdef __CUDA_ARCH__
  const double s = __dadd_rn(a, b);
  const double bb = __dsub_rn(s, a);
  const double err = __dadd_rn(__dsub_rn(a, __dsub_rn(s, bb)), __dsub_rn(b, bb));
#else
  const double s = a + b;
  const double bb = s - a;
  const double err = (a - (s - bb)) + (b - bb);
#endif
  return {s, err};
}

__host__ __device__ __forceinline__ Dd dd_add(Dd a, Dd b) {
  const Dd t = dd_two_sum(a.hi, b.hi);
#ifdef __CUDA_ARCH__
  const double lo = __dadd_rn(t.lo, __dadd_rn(a.lo, b.lo));
  const double hi = __dadd_rn(t.hi, lo);
  return {hi, __dsub_rn(lo, __dsub_rn(hi, t.hi))};
#else
  const double lo = t.lo + (a.lo + b.lo);
  const double hi = t.hi + lo;
  return {hi, lo - (hi - t.hi)};
#endif
}

__host__ __device__ __forceinline__ Dd dd_add(Dd acc, double x) {
  return dd_add(acc, Dd{x, 0.0});
}

__host__ __device__ __forceinline__ double dd_value(Dd a) {
#ifdef __CUDA_ARCH__
  return __dadd_rn(a.hi, a.lo);
#else
  return a.hi + a.lo;
#endif
}

// ---------------------------------------------------------------------------
// sm_90+/sm_100a async-copy + mbarrier primitives (inline PTX).

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(count)
               : "memory");
}

__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar,
                                                      uint32_t bytes) {
  asm volatile(
      "mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(
          smem_u32(bar)),
      "r"(bytes)
      : "memory");
}

// arrive from the threads where `pred` holds, without a divergent branch
__device__ __forceinline__ void mbar_arrive_if(uint64_t* bar, bool pred) {
  asm volatile(
      "{ .reg .pred p; setp.ne.u32 p, %1, 0; "
      "@p mbarrier.arrive.release.cta.shared::cta.b64 _, [%0]; }" ::"r"(smem_u32(bar)),
      "r"((uint32_t)pred)
      : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n"
      " mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\n"
      " selp.u32 %0, 1, 0, p;\n}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}

// L2 eviction-priority policies (createpolicy) for cache-hinted accesses
__device__ __forceinline__ uint64_t l2_policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t l2_policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// bulk copy global -> shared with an L2 cache policy (streaming data that
// should not displace data kept for a later kernel)
__device__ __forceinline__ void bulk_g2s_hint(void* dst, const void* src, uint32_t bytes,
                                              uint64_t* bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes.L2::cache_hint "
      "[%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}

// bulk prefetch of a global range into L2 (TMA engine; no completion)
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}

// store with an L2 cache policy
__device__ __forceinline__ void st_hint(double* p, double v, uint64_t policy) {
  asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(p), "d"(v), "l"(policy)
               : "memory");
}

// 1-D bulk copy global -> shared (TMA engine, no tensor map), completion
// counted in bytes on an mbarrier. dst/src 16-B aligned, bytes % 16 == 0.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src,
                                         uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], "
      "[%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// Make generic-proxy shared-memory writes visible to the async (TMA) proxy.
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// global[dst .. dst+bytes) += shared[src ..] element-wise (f64), by the TMA
// engine; completion tracked by the calling thread's bulk async-group.
__device__ __forceinline__ void bulk_reduce_add_f64(void* dst, const void* src,
                                                    uint32_t bytes) {
  asm volatile(
      "cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f64 [%0], [%1], "
      "%2;" ::"l"(dst),
      "r"(smem_u32(src)), "r"(bytes)
      : "memory");
}

__device__ __forceinline__ void bulk_commit_group() {
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}

// Wait until every committed bulk op of this thread has READ its source.
__device__ __forceinline__ void bulk_wait_group_read0() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}

__device__ __forceinline__ void named_bar_sync(int id, int threads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}

// Programmatic dependent launch (PDL): a kernel launched with
// launch_pdl() may start while its predecessor drains; pdl_wait() blocks until
// the predecessor grid has completed and its memory is visible, so it must
// precede every read of predecessor output (including CG's `done` flag).
__device__ __forceinline__ void pdl_wait() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
}
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) is per device: set it once
// per (call site, device); `mask` is the call site's static device bitmask.
template <typename Kernel>
inline cudaError_t smem_attr_once(Kernel* kernel, int bytes, std::atomic<uint64_t>& mask) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const uint64_t bit = 1ull << (dev & 63);
  if (mask.load(std::memory_order_acquire) & bit) return cudaSuccess;
  e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) mask.fetch_or(bit, std::memory_order_release);
  return e;
}

// Shared-memory carveout preference (percent of the maximum), once per device.
// A kernel meant to run beside a big-smem persistent kernel needs the SM
// configured for the full carveout, not the smallest one that fits.
template <typename Kernel>
inline cudaError_t carveout_once(Kernel* kernel, int pct, std::atomic<uint64_t>& mask) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const uint64_t bit = 1ull << (dev & 63);
  if (mask.load(std::memory_order_acquire) & bit) return cudaSuccess;
  e = cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout, pct);
  if (e == cudaSuccess) mask.fetch_or(bit, std::memory_order_release);
  return e;
}

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block,
                              size_t smem, cudaStream_t stream, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// launch_pdl with a 1-D thread-block cluster of `cluster` CTAs
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl_cluster(void (*kernel)(KArgs...), dim3 grid, dim3 block,
                                      int cluster, size_t smem, cudaStream_t stream,
                                      Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  attr[1].id = cudaLaunchAttributeClusterDimension;
  attr[1].val.clusterDim.x = (unsigned)cluster;
  attr[1].val.clusterDim.y = 1;
  attr[1].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

}  // namespace hs
