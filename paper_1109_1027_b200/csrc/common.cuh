// common.cuh — small device helpers for the sm_100a 2SHOC/RK4 kernels: complex arithmetic
// on interleaved (re, im) pairs, 128-bit vector moves, and the PTX wrappers for TMA
// (cp.async.bulk.tensor) and mbarriers.  Product code: shares nothing with oracle/.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <cstdio>

namespace nlse {

// Interleaved (re, im) pair with the alignment of the pair, so that one complex moves with
// one 8-byte (complex64) or 16-byte (complex128) access (fields are element-aligned).
template <typename R> struct alignas(2 * sizeof(R)) cplx { R re, im; };

template <typename R> __device__ __forceinline__ cplx<R> mk(R r, R i) { return {r, i}; }
template <typename R> __device__ __forceinline__ cplx<R> operator+(cplx<R> a, cplx<R> b) { return {a.re + b.re, a.im + b.im}; }
template <typename R> __device__ __forceinline__ cplx<R> operator-(cplx<R> a, cplx<R> b) { return {a.re - b.re, a.im - b.im}; }
template <typename R> __device__ __forceinline__ cplx<R> operator*(R s, cplx<R> a) { return {s * a.re, s * a.im}; }
// a + s*b with FMA
template <typename R> __device__ __forceinline__ cplx<R> axpy(cplx<R> a, R s, cplx<R> b) {
  return {fma(s, b.re, a.re), fma(s, b.im, a.im)};
}
template <typename R> __device__ __forceinline__ R norm2(cplx<R> a) { return fma(a.re, a.re, a.im * a.im); }
// a + s * (i t)  (the RK4 stage combine with F = i t)
template <typename R> __device__ __forceinline__ cplx<R> iaxpy(cplx<R> a, R s, cplx<R> t) {
  return {fma(-s, t.im, a.re), fma(s, t.re, a.im)};
}

// complex64: packed FP32x2 arithmetic (sm_100 FADD2 / FMUL2 / FFMA2 on the (re, im) pair),
// one instruction per complex operation instead of two.
__device__ __forceinline__ float2 f2(cplx<float> a) { return make_float2(a.re, a.im); }
__device__ __forceinline__ cplx<float> c2(float2 a) { return {a.x, a.y}; }
__device__ __forceinline__ cplx<float> operator+(cplx<float> a, cplx<float> b) { return c2(__fadd2_rn(f2(a), f2(b))); }
__device__ __forceinline__ cplx<float> operator-(cplx<float> a, cplx<float> b) {
  return c2(__ffma2_rn(f2(b), make_float2(-1.f, -1.f), f2(a)));
}
__device__ __forceinline__ cplx<float> operator*(float s, cplx<float> a) { return c2(__fmul2_rn(make_float2(s, s), f2(a))); }
__device__ __forceinline__ cplx<float> axpy(cplx<float> a, float s, cplx<float> b) {
  return c2(__ffma2_rn(f2(b), make_float2(s, s), f2(a)));
}
__device__ __forceinline__ cplx<float> iaxpy(cplx<float> a, float s, cplx<float> t) {
  return c2(__ffma2_rn(make_float2(t.im, t.re), make_float2(-s, s), f2(a)));
}

// ---------------------------------------------------------------------------------- PTX
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ bool mbar_try_wait(uint64_t *bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}

__device__ __forceinline__ bool mbar_try_wait_sleep(uint64_t *bar, uint32_t parity, uint32_t ns);
#ifdef NLSE_DEBUG_HANG
#define NLSE_HANG_CHECK(tag)                                                                              \
  if (++spins_ == (1u << 22))                                                                            \
    printf("hang? %s block %d thread %d bar %p parity %u\n", tag, blockIdx.x, threadIdx.x, (void *)bar, parity);
#else
#define NLSE_HANG_CHECK(tag)
#endif
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  if (mbar_try_wait(bar, parity)) return;  // fast path: phase already complete
  uint32_t spins_ = 0;
  (void)spins_;
  while (!mbar_try_wait_sleep(bar, parity, 20000)) {
    NLSE_HANG_CHECK("consumer")
  }
}

// Suspending wait: try_wait with a suspend-time hint parks the warp in hardware until the
// phase completes (or the hint expires) instead of spinning, so a waiting warp does not
// steal issue slots from the working warps of its scheduler.
__device__ __forceinline__ bool mbar_try_wait_sleep(uint64_t *bar, uint32_t parity, uint32_t ns) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2, %3;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity), "r"(ns)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait_backoff(uint64_t *bar, uint32_t parity) {
  uint32_t spins_ = 0;
  (void)spins_;
  while (!mbar_try_wait_sleep(bar, parity, 20000)) {
    NLSE_HANG_CHECK("producer")
  }
}

// 2D / 3D tiled TMA loads global -> shared with an L2 eviction-priority policy (createpolicy),
// completion counted on an mbarrier; e.g. evict_first for read-once streams so that the
// stencil input planes stay resident for neighbour halos.
__device__ __forceinline__ void tma_load_2d_hint(void *dst, const CUtensorMap *map, uint64_t *bar, int c0, int c1,
                                                 uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, "
      "%3}], [%4], %5;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d_hint(void *dst, const CUtensorMap *map, uint64_t *bar, int c0, int c1,
                                                 int c2, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, "
      "%3, %4}], [%5], %6;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
// Contiguous bulk copy global -> shared (one instruction for a whole row segment), completion
// counted on an mbarrier; bytes and both addresses multiples of 16.
__device__ __forceinline__ void bulk_load_hint(void *dst, const void *src, uint32_t bytes, uint64_t *bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}

__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_normal() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}

__device__ __forceinline__ void prefetch_tmap(const CUtensorMap *map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

// 128-bit global stores of the stage outputs (plain stores: evict-first / write-through
// variants measured no faster on C4 / C5W, profiles/r01/README.md)
__device__ __forceinline__ void st_stream(float4 *p, float4 v) { *p = v; }
__device__ __forceinline__ void st_stream(double2 *p, double2 v) { *p = v; }

// Checked build (-DNLSE_CHECKED, libnlse2shoc_checked.so; compute-sanitizer is not available
// on the GPU pool): every global store of the 2D/3D stage kernel is range-checked against
// the buffer it belongs to; a store outside is skipped and counted, and
// nlse2shoc_checked_violations() reads the count.  Normal builds compile the checks away.
#ifdef NLSE_CHECKED
__device__ unsigned long long g_nlse_violations;
// n elements of T at p lie inside [base, base + bytes)
template <typename T> __device__ __forceinline__ bool in_range(const T *p, int n, const void *base, int64_t bytes) {
  const char *b = reinterpret_cast<const char *>(base), *q = reinterpret_cast<const char *>(p);
  return base != nullptr && q >= b && q + int64_t(n) * int64_t(sizeof(T)) <= b + bytes;
}
#define NLSE_STORE_OK(p, n, base, bytes) (in_range((p), (n), (base), (bytes)) ? true : (atomicAdd(&g_nlse_violations, 1ull), false))
#else
#define NLSE_STORE_OK(p, n, base, bytes) true
#endif

// Fused halo exchange (stage_stream.cuh): wait until a counter that a neighbour slab raises
// with system-scope atomics reaches target, then order the halo reads that follow through the
// async proxy (TMA) after the acquire.
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long *p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
// The wait is bounded (~4 s): a neighbour that never arrives (a rank that died, or calls that
// differ between ranks) counts a timeout in *timeouts and lets the kernel finish instead of
// hanging the GPU; nlse2shoc_exchange_timeouts() reports it.
__device__ __forceinline__ void wait_counter(const unsigned long long *p, unsigned long long target,
                                             unsigned long long *timeouts) {
  uint32_t spins = 0;
  // once a wait has timed out on this slab, later ones do not wait (the call is invalid)
  while (ld_acquire_sys(p) < target && *reinterpret_cast<volatile unsigned long long *>(timeouts) == 0) {
    __nanosleep(128);
    if (++spins == (1u << 25)) {
      atomicAdd(timeouts, 1ull);
      break;
    }
  }
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

__device__ __forceinline__ void named_bar_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

}  // namespace nlse
