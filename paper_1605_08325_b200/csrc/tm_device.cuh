// Device-side building blocks shared by the sm_100a kernels of libtm.so:
// memory-ordering primitives for the cross-rank flags, 16-byte accesses, the
// binary16 conversions, status screening, the exact division by k, wire-unit
// traits, mbarrier / bulk-async (TMA engine) copy wrappers, and the elastic
// difference of EASGD.  Header-only; every function is inline.
#pragma once

#include <cuda_fp16.h>
#include <stdint.h>
#include <stdlib.h>

#include <algorithm>
#include <atomic>

#include "tm_internal.h"

namespace tmx {

// ------------------------------------------------------------ host helpers
inline int sm_count(int device) {
  int n = 0;
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device);
  return n > 0 ? n : 1;
}

inline int env_int(const char* name, int dflt) {
  const char* v = getenv(name);
  return (v && *v) ? atoi(v) : dflt;
}

// Opt kernel `fn` into `bytes` of dynamic shared memory on device `dev`, once
// per (kernel, device): `done` is the caller's per-kernel bit set of devices.
inline cudaError_t smem_optin(const void* fn, int bytes, int dev, std::atomic<uint64_t>& done) {
  const uint64_t bit = 1ull << (dev & 63);
  if (done.load(std::memory_order_acquire) & bit) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) done.fetch_or(bit, std::memory_order_release);
  return e;
}

// grid for a grid-stride streaming kernel over `work_items` thread-items
inline int streaming_grid(int64_t work_items) {
  int dev = 0;
  cudaGetDevice(&dev);
  int64_t want = (work_items + kThreads - 1) / kThreads;
  return (int)std::min<int64_t>(std::max<int64_t>(want, 1), 4 * sm_count(dev));
}

namespace dev {

__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// GPU-scope versions: enough when every rank of the exchange runs on this GPU
// (a single-process group), where system scope would only add fence cost.
__device__ __forceinline__ void st_release_gpu(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_gpu(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

template <bool SYS>
__device__ __forceinline__ void st_release(uint32_t* p, uint32_t v) {
  if constexpr (SYS) st_release_sys(p, v);
  else st_release_gpu(p, v);
}
template <bool SYS>
__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* p) {
  if constexpr (SYS) return ld_acquire_sys(p);
  else return ld_acquire_gpu(p);
}

// 16-byte accesses.  Peer / staging data is written during the same kernel by
// other SMs or GPUs, so the non-coherent (.nc) path is never used for it; .cg
// caches in L2 only.
__device__ __forceinline__ uint4 ld16_cg(const void* p) {
  return __ldcg(reinterpret_cast<const uint4*>(p));
}
__device__ __forceinline__ void st16_cg(void* p, uint4 v) {
  __stcg(reinterpret_cast<uint4*>(p), v);
}
__device__ __forceinline__ float4 ld16_f(const float* p) {
  return __ldcs(reinterpret_cast<const float4*>(p));
}
__device__ __forceinline__ void st16_f(float* p, float4 v) {
  __stcs(reinterpret_cast<float4*>(p), v);
}

__device__ __forceinline__ uint32_t pack_rn16x2(float lo, float hi) {
  __half2 h = __floats2half2_rn(lo, hi);  // cvt.rn.f16x2.f32
  return *reinterpret_cast<uint32_t*>(&h);
}
__device__ __forceinline__ float2 unpack16x2(uint32_t u) {
  __half2 h = *reinterpret_cast<__half2*>(&u);
  return __half22float2(h);  // exact
}

// Status bits of one fp32 value: non-finite; |x| >= 65520 (rounds to fp16 inf).
__device__ __forceinline__ uint32_t status_of(float v, bool wire16) {
  const uint32_t b = __float_as_uint(v) & 0x7fffffffu;
  uint32_t s = (b >= 0x7f800000u) ? TM_BIT_NONFINITE : 0u;
  if (wire16 && b < 0x7f800000u && b >= 0x477ff000u) s |= TM_BIT_OVERFLOW16;  // 65520.0f
  return s;
}

// fl(s / k).  For k a power of two the product with the exact 1/k is the same
// correctly rounded value (x/2^n and x*2^-n are the same real number), and is
// cheaper; otherwise an IEEE division.
template <int K>
__device__ __forceinline__ float div_k(float s) {
  if constexpr ((K & (K - 1)) == 0) return __fmul_rn(s, 1.0f / (float)K);
  else return __fdiv_rn(s, (float)K);
}

// Status of a unit of E fp32 values: a max over |bits| screens the unit (one
// LOP + one IMNMX per element); the exact bits are computed only when the max
// reaches the fp16-overflow (ASA16) or non-finite (ASA) threshold.
template <bool W16, int E>
__device__ __forceinline__ uint32_t unit_status(const float* f) {
  uint32_t m = 0;
#pragma unroll
  for (int q = 0; q < E; ++q) m = max(m, __float_as_uint(f[q]) & 0x7fffffffu);
  if (m < (W16 ? 0x477ff000u : 0x7f800000u)) return 0u;
  uint32_t st = 0;
#pragma unroll
  for (int q = 0; q < E; ++q) st |= status_of(f[q], W16);
  return st;
}

// ---------------------------------------------------------------------------
// Wire-type traits: one "unit" = 16 bytes of wire data.
//   fp16 wire: 8 elements (32 B of fp32 source);  fp32 wire: 4 elements.
// ---------------------------------------------------------------------------
template <bool W16>
struct Unit;

template <>
struct Unit<true> {
  static constexpr int kElems = 8;
  struct Src { float4 a, b; };
  __device__ static Src load_src(const float* p) { return {ld16_f(p), ld16_f(p + 4)}; }
  __device__ static void to_floats(const Src& s, float* f) {
    f[0] = s.a.x; f[1] = s.a.y; f[2] = s.a.z; f[3] = s.a.w;
    f[4] = s.b.x; f[5] = s.b.y; f[6] = s.b.z; f[7] = s.b.w;
  }
  __device__ static uint4 encode(const float* f) {
    return make_uint4(pack_rn16x2(f[0], f[1]), pack_rn16x2(f[2], f[3]),
                      pack_rn16x2(f[4], f[5]), pack_rn16x2(f[6], f[7]));
  }
  __device__ static void decode(uint4 u, float* f) {
    float2 t;
    t = unpack16x2(u.x); f[0] = t.x; f[1] = t.y;
    t = unpack16x2(u.y); f[2] = t.x; f[3] = t.y;
    t = unpack16x2(u.z); f[4] = t.x; f[5] = t.y;
    t = unpack16x2(u.w); f[6] = t.x; f[7] = t.y;
  }
  __device__ static void store_dst(float* p, const float* f) {
    st16_f(p, make_float4(f[0], f[1], f[2], f[3]));
    st16_f(p + 4, make_float4(f[4], f[5], f[6], f[7]));
  }
};

template <>
struct Unit<false> {
  static constexpr int kElems = 4;
  struct Src { float4 a; };
  __device__ static Src load_src(const float* p) { return {ld16_f(p)}; }
  __device__ static void to_floats(const Src& s, float* f) {
    f[0] = s.a.x; f[1] = s.a.y; f[2] = s.a.z; f[3] = s.a.w;
  }
  __device__ static uint4 encode(const float* f) {
    return make_uint4(__float_as_uint(f[0]), __float_as_uint(f[1]), __float_as_uint(f[2]),
                      __float_as_uint(f[3]));
  }
  __device__ static void decode(uint4 u, float* f) {
    f[0] = __uint_as_float(u.x); f[1] = __uint_as_float(u.y);
    f[2] = __uint_as_float(u.z); f[3] = __uint_as_float(u.w);
  }
  __device__ static void store_dst(float* p, const float* f) {
    st16_f(p, make_float4(f[0], f[1], f[2], f[3]));
  }
};

// fp16 round trip of 4 values: widen(rn16(v)) (ASA16 quantisation, reading R1)
__device__ __forceinline__ float4 q16(float4 v) {
  const float2 lo = unpack16x2(pack_rn16x2(v.x, v.y));
  const float2 hi = unpack16x2(pack_rn16x2(v.z, v.w));
  return make_float4(lo.x, lo.y, hi.x, hi.y);
}

// Momentum-SGD step of 4 elements (one IEEE rounding per operation,
// no FMA): v' = fl(fl(mu*v) - fl(lr*g)); the weights then take w' = fl(w + v').
__device__ __forceinline__ float4 sgd_v(float4 v, float4 g, float lr, float mu) {
  return make_float4(__fsub_rn(__fmul_rn(mu, v.x), __fmul_rn(lr, g.x)),
                     __fsub_rn(__fmul_rn(mu, v.y), __fmul_rn(lr, g.y)),
                     __fsub_rn(__fmul_rn(mu, v.z), __fmul_rn(lr, g.z)),
                     __fsub_rn(__fmul_rn(mu, v.w), __fmul_rn(lr, g.w)));
}
__device__ __forceinline__ float sgd_v1(float v, float g, float lr, float mu) {
  return __fsub_rn(__fmul_rn(mu, v), __fmul_rn(lr, g));
}
__device__ __forceinline__ float4 add4(float4 a, float4 b) {
  return make_float4(__fadd_rn(a.x, b.x), __fadd_rn(a.y, b.y), __fadd_rn(a.z, b.z), __fadd_rn(a.w, b.w));
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
// Upper bound on the depth of every bulk-copy ring; the mbarrier arrays are
// declared with this many slots (see easgd_round_tma_kernel).
constexpr int kMaxStages = 8;

// Dynamic tile claiming without a host-side reset: ctr[0] is the claim counter
// of the launch, ctr[1] counts CTAs that have made their last claim.  Thread 0
// calls this once its CTA will claim no more; the last CTA to retire resets both
// words for the next launch (the kernel boundary orders the reset before it).
// Both words start at zero (the library's slab is zeroed at init).
__device__ __forceinline__ void tile_ctr_retire(unsigned long long* ctr) {
  __threadfence();  // this CTA's claims precede its retirement
  if (atomicAdd(ctr + 1, 1ull) == (unsigned long long)gridDim.x - 1) {
    ctr[0] = 0;
    ctr[1] = 0;
  }
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)), "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_load(void* smem_dst, const void* gmem_src, uint32_t bytes,
                                          uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(smem_dst)),
      "l"(gmem_src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// The same mbarrier operations on a precomputed 32-bit shared address (one
// address computation per barrier array, reused by every operation on it).
__device__ __forceinline__ void mbar_init_a(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx_a(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait_a(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(bar), "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_load_a(void* smem_dst, const void* gmem_src, uint32_t bytes, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(smem_dst)),
      "l"(gmem_src), "r"(bytes), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void bulk_store(void* gmem_dst, const void* smem_src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gmem_dst),
               "r"(smem_u32(smem_src)), "r"(bytes)
               : "memory");
}
// L2 eviction-priority variants (A/B knob TM_L2_HINT of the direct kernel): the
// policy comes from createpolicy; streamed-once data may be marked evict_first.
__device__ __forceinline__ uint64_t l2_policy_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void bulk_load_hint(void* smem_dst, const void* gmem_src, uint32_t bytes,
                                               uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::
          "r"(smem_u32(smem_dst)),
      "l"(gmem_src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void bulk_store_hint(void* gmem_dst, const void* smem_src, uint32_t bytes,
                                                uint64_t pol) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(gmem_dst),
               "r"(smem_u32(smem_src)), "r"(bytes), "l"(pol)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait_all() {
  asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ float elastic_diff(float x, float c, float alpha) {
  return __fmul_rn(alpha, __fsub_rn(x, c));
}

__device__ __forceinline__ void red_add_sys(float* p, float v) {
  asm volatile("red.relaxed.sys.global.add.f32 [%0], %1;" ::"l"(p), "f"(v) : "memory");
}

__device__ __forceinline__ void red_add_gpu(float* p, float v) {
  asm volatile("red.relaxed.gpu.global.add.f32 [%0], %1;" ::"l"(p), "f"(v) : "memory");
}

// Four independent fp32 atomic adds in one instruction (sm_90+ vector red; each
// element's add is atomic on its own, exactly as four scalar reds).  p 16-B aligned.
__device__ __forceinline__ void red_add4_sys(float* p, float4 v) {
  asm volatile("red.relaxed.sys.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(v.x), "f"(v.y),
               "f"(v.z), "f"(v.w)
               : "memory");
}
__device__ __forceinline__ void red_add4_gpu(float* p, float4 v) {
  asm volatile("red.relaxed.gpu.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(v.x), "f"(v.y),
               "f"(v.z), "f"(v.w)
               : "memory");
}

}  // namespace dev
}  // namespace tmx
