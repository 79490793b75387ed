// sm_100a kernels of the Theano-MPI parameter exchange (arXiv 1605.08325).
//
//   tm_exchange_kernel  -- ASA / ASA16: one persistent,
//                          cooperative launch per exchange, three phases per CTA
//                          separated by cross-rank per-CTA epoch flags:
//        a2 pre-cast   x (fp32, caller's buffer) -> stage (wire type), all k
//                      segments of this CTA's chunk; rn16 for ASA16 (reading R1:
//                      the own segment is rounded too); non-finite / fp16
//                      overflow detection fused.
//        a3 ready barrier.
//        a4 reduce-scatter PULL: for the own segment r, load the chunk from every
//                      rank's stage (peer pointers: NVLink P2P loads on a real box,
//                      local HBM in a single-process group), widen, sum in
//                      ascending rank from the rank-0 term, one IEEE division by
//                      k, round to the wire type, store to the own `avg`.
//        a5 reduced barrier.
//        a6 allgather PULL: load every rank's `avg` chunk, widen, store into the
//                      caller's buffer (truncated at P).
//   local_allreduce     -- AR when all k ranks live in this process: one pass.
//   easgd / easgd_round -- elastic update.
//   cast_rn16           -- test hook: the device rounding used by a2/a4.
//
// Numerics: every fp32 op is an explicit round-to-nearest intrinsic
// (__fadd_rn/__fsub_rn/__fmul_rn/__fdiv_rn: no FMA contraction, IEEE division);
// the library is compiled without --use_fast_math (no FTZ).  The binary16
// conversions are cvt.rn.f16(x2).f32 (RNE, gradual subnormals, overflow to inf)
// and the exact cvt.f32.f16.
//
// Memory-ordering protocol (a3/a5): after __syncthreads(), thread j < k writes
// the epoch into rank j's flag slot [phase][r][c] with st.release.sys and then
// spins with ld.acquire.sys on its own slot [phase][j][c]; a second
// __syncthreads() publishes the acquisition to the CTA.  Flags only couple CTA
// c of every rank, so no grid-wide barrier is needed.  Reuse of stage/avg across
// back-to-back exchanges is safe without a trailing barrier:
//   stage_j(n+1) is written only after rank j saw REDUCED(n) from every rank,
//     i.e. after every rank finished reading stage_j(n);
//   avg_j(n+1) is written only after rank j saw READY(n+1) from every rank, which
//     each rank signals after its AG(n) reads of avg_j(n).

#include <cuda_fp16.h>
#include <stdint.h>

#include <stdlib.h>

#include <algorithm>

#include "tm_internal.h"

namespace tmx {
namespace {

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

// Cross-rank, per-CTA epoch barrier (see the protocol in the file header).
// Returns false (whole CTA) if a peer timed out.
template <int K, bool SYS>
__device__ __forceinline__ bool rank_barrier(const ExchangeArgs& a, int phase, int r, int c,
                                             uint32_t epoch, int* s_abort) {
  __syncthreads();
  if (threadIdx.x < K) {
    const int j = threadIdx.x;
    uint32_t* remote = a.flags[j] + (size_t)(phase * TM_MAX_RANKS + r) * a.C + c;
    st_release<SYS>(remote, epoch);
    const uint32_t* mine = a.flags[r] + (size_t)(phase * TM_MAX_RANKS + j) * a.C + c;
    if ((int32_t)(ld_acquire<SYS>(mine) - epoch) < 0) {
      const uint64_t t0 = globaltimer();
      while ((int32_t)(ld_acquire<SYS>(mine) - epoch) < 0) {
        if (globaltimer() - t0 > a.timeout_ns) {
          atomicOr(a.status, TM_BIT_TIMEOUT);
          *s_abort = 1;
          break;
        }
        __nanosleep(32);
      }
    }
  }
  __syncthreads();
  return *s_abort == 0;
}

template <int K, bool W16, bool SYS>
__global__ void __launch_bounds__(kThreads, K == 6 ? 3 : 4)
tm_exchange_kernel(const __grid_constant__ ExchangeArgs a) {
  using U = Unit<W16>;
  constexpr int E = U::kElems;
  constexpr int WB = W16 ? 2 : 4;  // wire bytes per element
  __shared__ int s_abort;
  __shared__ uint32_t s_epoch;

  const int lr = blockIdx.x / a.C;
  const int c = blockIdx.x - lr * a.C;
  const int r = a.rank0 + lr;
  // Device-side epoch: CTA c of rank r owns counter ctr[c] in its own flag pad
  // (after the [kPhases][TM_MAX_RANKS][C] slots).  Every rank performs the same
  // sequence of exchanges, so the counters advance in lockstep; keeping the
  // epoch on the device leaves the launch parameters constant across calls,
  // which makes the exchange capturable in a CUDA graph.
  if (threadIdx.x == 0) {
    s_abort = 0;
    uint32_t* ctr = a.flags[r] + (size_t)kPhases * TM_MAX_RANKS * a.C + c;
    s_epoch = *ctr + 1;
    *ctr = s_epoch;
  }
  __syncthreads();
  const uint32_t epoch = s_epoch;
  float* __restrict__ x = a.x[lr];
  const int64_t P = a.P, L = a.L;
  const int64_t e0 = (int64_t)c * a.Lc;
  const int64_t e1 = min(e0 + a.Lc, L);
  const int64_t nu = e1 > e0 ? (e1 - e0) / E : 0;  // wire units per segment chunk
  char* const stage_r = reinterpret_cast<char*>(a.stage[r]);

  // ---------------- a2: pre-cast all k segments' chunk c into own stage -------
  // Thread-contiguous units within a segment (coalesced); G segments per batch
  // so G independent 32-byte (ASA16) / 16-byte (ASA) loads are in flight.
  const int nu32 = (int)nu;
  uint32_t st = 0;
  {
    constexpr int G = K < 4 ? K : 4;
    for (int v = threadIdx.x; v < nu32; v += kThreads) {
      const int64_t ev = e0 + (int64_t)v * E;
#pragma unroll
      for (int s0 = 0; s0 < K; s0 += G) {
        float f[G][E];
#pragma unroll
        for (int u = 0; u < G; ++u) {
          if (s0 + u < K) {
            const int64_t g = (int64_t)(s0 + u) * L + ev;
            if (g + E <= P) {
              U::to_floats(U::load_src(x + g), f[u]);
            } else {
#pragma unroll
              for (int q = 0; q < E; ++q) f[u][q] = (g + q < P) ? x[g + q] : 0.0f;
            }
          }
        }
#pragma unroll
        for (int u = 0; u < G; ++u) {
          if (s0 + u < K) {
            const int64_t g = (int64_t)(s0 + u) * L + ev;
            st |= unit_status<W16, E>(f[u]);
            st16_cg(stage_r + g * WB, U::encode(f[u]));
          }
        }
      }
    }
  }
  if (st) atomicOr(a.status, st);  // rare: only threads that saw a bad value

  if (!rank_barrier<K, SYS>(a, kPhaseReady, r, c, epoch, &s_abort)) return;

  // ---------------- a4: reduce-scatter pull, fused sum / (1/k) / cast -------
  {
    const char* src[K];
#pragma unroll
    for (int j = 0; j < K; ++j) src[j] = reinterpret_cast<const char*>(a.stage[j]);
    char* const avg_r = reinterpret_cast<char*>(a.avg[r]);
    const int64_t seg0 = (int64_t)r * L + e0;
    for (int64_t v = threadIdx.x; v < nu; v += kThreads) {
      const int64_t off = (seg0 + v * E) * WB;
      uint4 raw[K];
#pragma unroll
      for (int j = 0; j < K; ++j) raw[j] = ld16_cg(src[j] + off);
      float s[E], t[E];
      U::decode(raw[0], s);
#pragma unroll
      for (int j = 1; j < K; ++j) {
        U::decode(raw[j], t);
#pragma unroll
        for (int q = 0; q < E; ++q) s[q] = __fadd_rn(s[q], t[q]);
      }
#pragma unroll
      for (int q = 0; q < E; ++q) s[q] = div_k<K>(s[q]);
      st16_cg(avg_r + (e0 + v * E) * WB, U::encode(s));
    }
  }

  if (!rank_barrier<K, SYS>(a, kPhaseReduced, r, c, epoch, &s_abort)) return;

  // ---------------- a6: allgather pull, fused widen, store to caller ---------
  {
    constexpr int G = K;  // all k owners' units in flight at once
    for (int v = threadIdx.x; v < nu32; v += kThreads) {
      const int64_t ev = e0 + (int64_t)v * E;
      uint4 raw[G];
#pragma unroll
      for (int j = 0; j < G; ++j)
        raw[j] = ld16_cg(reinterpret_cast<const char*>(a.avg[j]) + ev * WB);
#pragma unroll
      for (int j = 0; j < G; ++j) {
        const int64_t g = (int64_t)j * L + ev;
        float f[E];
        U::decode(raw[j], f);
        if (g + E <= P) {
          U::store_dst(x + g, f);
        } else {
#pragma unroll
          for (int q = 0; q < E; ++q)
            if (g + q < P) x[g + q] = f[q];
        }
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Single-process group, one pass ("direct" path).  When all k ranks' buffers
// are addressable by one kernel there is no wire: the owner of each element
// pulls the k contributions straight from the k buffers (the Alltoall leg),
// applies the method's arithmetic in registers -- rn16 of every contribution
// (ASA16, reading R1), ascending-rank fp32 sum from the rank-0 term, fl(s/k),
// rn16 of the average -- and pushes widen(result) into all k buffers (the
// Allgather leg).  Element i is read and written only by the thread that owns
// it, so no flags are needed; the kernel boundary orders consecutive
// exchanges.  Results are bitwise those of the staged path (elementwise
// method, readings Q7/Q9).  Also AR for a single-process group (Q16 = false).
// ---------------------------------------------------------------------------
struct LocalBufs {
  float* b[TM_MAX_RANKS];
};

__device__ __forceinline__ float4 q16(float4 v) {
  const float2 lo = unpack16x2(pack_rn16x2(v.x, v.y));
  const float2 hi = unpack16x2(pack_rn16x2(v.z, v.w));
  return make_float4(lo.x, lo.y, hi.x, hi.y);
}

// The method's arithmetic on 4 elements of k contributions (registers in, one
// float4 out): rn16 of each contribution (Q16), ascending-rank sum from the
// rank-0 term, fl(s/k), rn16 of the average.  `st` accumulates status bits.
template <int K, bool Q16>
__device__ __forceinline__ float4 average4(const float4 (&in)[K], uint32_t& st) {
  // running max of |bits| screens for non-finite / fp16-overflow inputs
  uint32_t m = max(max(__float_as_uint(in[0].x) & 0x7fffffffu, __float_as_uint(in[0].y) & 0x7fffffffu),
                   max(__float_as_uint(in[0].z) & 0x7fffffffu, __float_as_uint(in[0].w) & 0x7fffffffu));
  float4 s = Q16 ? q16(in[0]) : in[0];
#pragma unroll
  for (int j = 1; j < K; ++j) {
    m = max(m, max(max(__float_as_uint(in[j].x) & 0x7fffffffu, __float_as_uint(in[j].y) & 0x7fffffffu),
                   max(__float_as_uint(in[j].z) & 0x7fffffffu, __float_as_uint(in[j].w) & 0x7fffffffu)));
    const float4 t = Q16 ? q16(in[j]) : in[j];
    s.x = __fadd_rn(s.x, t.x); s.y = __fadd_rn(s.y, t.y);
    s.z = __fadd_rn(s.z, t.z); s.w = __fadd_rn(s.w, t.w);
  }
  if (m >= (Q16 ? 0x477ff000u : 0x7f800000u)) {  // rare: exact bits from the inputs
#pragma unroll
    for (int j = 0; j < K; ++j)
      st |= status_of(in[j].x, Q16) | status_of(in[j].y, Q16) | status_of(in[j].z, Q16) |
            status_of(in[j].w, Q16);
  }
  s.x = div_k<K>(s.x); s.y = div_k<K>(s.y); s.z = div_k<K>(s.z); s.w = div_k<K>(s.w);
  if (Q16) s = q16(s);
  return s;
}

// Scalar version for the last P % 4 elements.
template <int K, bool Q16>
__device__ __forceinline__ void average1(const LocalBufs& lb, int64_t i, uint32_t& st) {
  float in[K];
#pragma unroll
  for (int j = 0; j < K; ++j) in[j] = lb.b[j][i];
#pragma unroll
  for (int j = 0; j < K; ++j) st |= status_of(in[j], Q16);
  float s = Q16 ? __half2float(__float2half_rn(in[0])) : in[0];
#pragma unroll
  for (int j = 1; j < K; ++j) s = __fadd_rn(s, Q16 ? __half2float(__float2half_rn(in[j])) : in[j]);
  s = div_k<K>(s);
  if (Q16) s = __half2float(__float2half_rn(s));
#pragma unroll
  for (int j = 0; j < K; ++j) lb.b[j][i] = s;
}

// Register-staged variant (16-byte LDG/STG, grid-stride over [e_begin, P)).
template <int K, bool Q16>
__global__ void __launch_bounds__(kThreads, K >= 7 ? 3 : 4)
tm_direct_kernel(const __grid_constant__ LocalBufs lb, int64_t e_begin, int64_t P,
                 uint32_t* status) {
  const int64_t v0 = e_begin / 4, nv = P / 4;
  const int64_t stride = (int64_t)gridDim.x * kThreads;
  uint32_t st = 0;
  for (int64_t v = v0 + (int64_t)blockIdx.x * kThreads + threadIdx.x; v < nv; v += stride) {
    float4 in[K];
#pragma unroll
    for (int j = 0; j < K; ++j) in[j] = ld16_f(lb.b[j] + v * 4);
    const float4 s = average4<K, Q16>(in, st);
#pragma unroll
    for (int j = 0; j < K; ++j) st16_f(lb.b[j] + v * 4, s);
  }
  const int64_t i = nv * 4 + threadIdx.x;  // tail (P % 4 elements), scalar
  if (blockIdx.x == 0 && i < P) average1<K, Q16>(lb, i, st);
  if (st) atomicOr(status, st);
}

// ---------------------------------------------------------------------------
// Bulk-async (TMA engine) variant of the direct path.  Persistent: one CTA per
// SM walks tiles of kTile elements.  Thread 0 streams each tile of all k
// buffers into a kStages-deep shared-memory ring with cp.async.bulk (1-D bulk
// copies completing on an mbarrier with expect_tx), every thread averages 4
// elements from shared memory, writes the result tile once to a small output
// ring, and thread 0 bulk-stores it into all k buffers
// (cp.async.bulk.global.shared::cta).  Bytes in flight are set by the ring
// depth, not by registers or LSU instruction count.  Elements past the last
// whole tile go through the register path above (same arithmetic).
// ---------------------------------------------------------------------------
constexpr int kOutRing = 4;  // output tiles in flight

// TILE: elements per buffer per tile; RING_KB: input ring budget; MINB: CTAs per SM.
template <int K, int TILE, int RING_KB, int MINB>
struct TmaCfg {
  static constexpr int kTileBytes = TILE * 4;
  static constexpr int kStagesRaw = RING_KB * 1024 / (K * kTileBytes);
  static constexpr int kStages = kStagesRaw > 8 ? 8 : (kStagesRaw < 2 ? 2 : kStagesRaw);
  static constexpr int kSmem = kStages * K * kTileBytes + kOutRing * kTileBytes;
  static constexpr int kVecPerThread = TILE / (4 * kThreads);
  static_assert(TILE % (4 * kThreads) == 0, "whole float4s per thread");
};

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
__device__ __forceinline__ void bulk_store(void* gmem_dst, const void* smem_src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gmem_dst),
               "r"(smem_u32(smem_src)), "r"(bytes)
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

template <int K, bool Q16, int TILE, int RING_KB, int MINB>
__global__ void __launch_bounds__(kThreads, MINB)
tm_direct_tma_kernel(const __grid_constant__ LocalBufs lb, int64_t ntiles, int64_t P,
                     uint32_t* status) {
  using Cfg = TmaCfg<K, TILE, RING_KB, MINB>;
  constexpr int S = Cfg::kStages;
  constexpr int V = Cfg::kVecPerThread;
  constexpr uint32_t TB = Cfg::kTileBytes;
  extern __shared__ __align__(128) unsigned char smem[];
  float* ring = reinterpret_cast<float*>(smem);                  // [S][K][TILE]
  float* outr = ring + (size_t)S * K * TILE;                     // [kOutRing][TILE]
  __shared__ __align__(8) uint64_t full[S];

  const int tid = threadIdx.x;
  // tiles of this CTA: blockIdx.x, blockIdx.x + gridDim.x, ...
  const int64_t my = blockIdx.x < ntiles ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  auto tile_of = [&](int64_t i) { return (int64_t)blockIdx.x + i * gridDim.x; };
  auto issue = [&](int64_t i) {
    const int s = (int)(i % S);
    const int64_t t = tile_of(i);
    mbar_expect_tx(&full[s], K * TB);
#pragma unroll
    for (int j = 0; j < K; ++j)
      bulk_load(ring + ((size_t)s * K + j) * TILE, lb.b[j] + t * TILE, TB, &full[s]);
  };

  if (tid == 0) {
    for (int s = 0; s < S; ++s) mbar_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int64_t i = 0; i < S && i < my; ++i) issue(i);
  }
  __syncthreads();

  uint32_t st = 0;
  for (int64_t i = 0; i < my; ++i) {
    const int s = (int)(i % S);
    mbar_wait(&full[s], (uint32_t)((i / S) & 1));
    float* out = outr + (size_t)(i % kOutRing) * TILE;
#pragma unroll
    for (int u = 0; u < V; ++u) {
      float4 in[K];
#pragma unroll
      for (int j = 0; j < K; ++j)
        in[j] = reinterpret_cast<const float4*>(ring + ((size_t)s * K + j) * TILE)[tid + u * kThreads];
      reinterpret_cast<float4*>(out)[tid + u * kThreads] = average4<K, Q16>(in, st);
    }
    fence_proxy_async_smem();  // generic-proxy smem writes -> visible to the bulk store
    if (tid == 0) bulk_wait_read<kOutRing - 2>();  // out slot of tile i+1 is free
    __syncthreads();
    if (tid == 0) {
      const int64_t t = tile_of(i);
#pragma unroll
      for (int j = 0; j < K; ++j) bulk_store(lb.b[j] + t * TILE, out, TB);
      bulk_commit();
      if (i + S < my) issue(i + S);  // every thread has finished reading ring slot s
    }
  }
  if (tid == 0) bulk_wait_all<0>();

  // elements past the last whole tile: register path (one CTA)
  if (blockIdx.x == gridDim.x - 1) {
    const int64_t e0 = ntiles * TILE;
    for (int64_t v = e0 / 4 + tid; v < P / 4; v += kThreads) {
      float4 in[K];
#pragma unroll
      for (int j = 0; j < K; ++j) in[j] = ld16_f(lb.b[j] + v * 4);
      const float4 r = average4<K, Q16>(in, st);
#pragma unroll
      for (int j = 0; j < K; ++j) st16_f(lb.b[j] + v * 4, r);
    }
    const int64_t i = (P / 4) * 4 + tid;
    if (i < P) average1<K, Q16>(lb, i, st);
  }
  if (st) atomicOr(status, st);
}

// ---------------------------------------------------------------------------
// EASGD elastic update, one fp32 op per step:
//   d = fl(x - c); e = fl(alpha d); x' = fl(x - e); c' = fl(c + e).
// Concurrent mode applies c += e with red.relaxed.sys.global.add.f32 so several
// workers (possibly on other GPUs, through an IPC mapping) may update one
// centre at once without lost updates; each worker then read a possibly stale c.
// ---------------------------------------------------------------------------
__device__ __forceinline__ float elastic_diff(float x, float c, float alpha) {
  return __fmul_rn(alpha, __fsub_rn(x, c));
}

__device__ __forceinline__ void red_add_sys(float* p, float v) {
  asm volatile("red.relaxed.sys.global.add.f32 [%0], %1;" ::"l"(p), "f"(v) : "memory");
}

template <bool Concurrent>
__global__ void __launch_bounds__(kThreads)
easgd_kernel(float* __restrict__ x, float* c, int64_t n, float alpha, int vec) {
  const int64_t stride = (int64_t)gridDim.x * kThreads;
  const int64_t tid = (int64_t)blockIdx.x * kThreads + threadIdx.x;
  int64_t done = 0;
  if (vec) {
    const int64_t nv = n / 4;
    for (int64_t v = tid; v < nv; v += stride) {
      float4 xv = ld16_f(x + v * 4);
      float4 cv = Concurrent ? __ldcg(reinterpret_cast<const float4*>(c + v * 4))
                             : ld16_f(c + v * 4);
      const float ex = elastic_diff(xv.x, cv.x, alpha), ey = elastic_diff(xv.y, cv.y, alpha);
      const float ez = elastic_diff(xv.z, cv.z, alpha), ew = elastic_diff(xv.w, cv.w, alpha);
      xv.x = __fsub_rn(xv.x, ex); xv.y = __fsub_rn(xv.y, ey);
      xv.z = __fsub_rn(xv.z, ez); xv.w = __fsub_rn(xv.w, ew);
      st16_f(x + v * 4, xv);
      if (Concurrent) {
        float* cp = c + v * 4;
        red_add_sys(cp, ex); red_add_sys(cp + 1, ey);
        red_add_sys(cp + 2, ez); red_add_sys(cp + 3, ew);
      } else {
        cv.x = __fadd_rn(cv.x, ex); cv.y = __fadd_rn(cv.y, ey);
        cv.z = __fadd_rn(cv.z, ez); cv.w = __fadd_rn(cv.w, ew);
        st16_f(c + v * 4, cv);
      }
    }
    done = nv * 4;
  }
  for (int64_t i = done + tid; i < n; i += stride) {
    const float xi = x[i];
    const float ci = Concurrent ? __ldcg(c + i) : c[i];
    const float e = elastic_diff(xi, ci, alpha);
    x[i] = __fsub_rn(xi, e);
    if (Concurrent) red_add_sys(c + i, e);
    else c[i] = __fadd_rn(ci, e);
  }
}

// Elastic update against a centre sharded by segment: element i
// of segment s = i / L lives at shard[s][i - s*L], local or on peer s over NVLink.
// Segments are multiples of 256 elements, so a 16-byte vector never straddles
// two shards.  Concurrent mode: c += e by red.add at system scope when the
// shard may be on another GPU.
__device__ __forceinline__ void red_add_gpu(float* p, float v) {
  asm volatile("red.relaxed.gpu.global.add.f32 [%0], %1;" ::"l"(p), "f"(v) : "memory");
}

template <bool Concurrent, bool SYS>
__global__ void __launch_bounds__(kThreads)
easgd_sharded_kernel(float* __restrict__ x, const __grid_constant__ ShardArgs sa, float alpha) {
  const int64_t stride = (int64_t)gridDim.x * kThreads;
  const int64_t tid = (int64_t)blockIdx.x * kThreads + threadIdx.x;
  for (int s = 0; s < sa.k; ++s) {
    const int64_t base = (int64_t)s * sa.L;
    const int64_t len = min(sa.L, sa.P - base);
    if (len <= 0) break;
    float* c = sa.shard[s];
    float* xs = x + base;
    const int64_t nv = len / 4;
    for (int64_t v = tid; v < nv; v += stride) {
      float4 xv = ld16_f(xs + v * 4);
      float4 cv = __ldcg(reinterpret_cast<const float4*>(c + v * 4));
      const float ex = elastic_diff(xv.x, cv.x, alpha), ey = elastic_diff(xv.y, cv.y, alpha);
      const float ez = elastic_diff(xv.z, cv.z, alpha), ew = elastic_diff(xv.w, cv.w, alpha);
      xv.x = __fsub_rn(xv.x, ex); xv.y = __fsub_rn(xv.y, ey);
      xv.z = __fsub_rn(xv.z, ez); xv.w = __fsub_rn(xv.w, ew);
      st16_f(xs + v * 4, xv);
      if (Concurrent) {
        float* cp = c + v * 4;
        if (SYS) { red_add_sys(cp, ex); red_add_sys(cp + 1, ey); red_add_sys(cp + 2, ez); red_add_sys(cp + 3, ew); }
        else { red_add_gpu(cp, ex); red_add_gpu(cp + 1, ey); red_add_gpu(cp + 2, ez); red_add_gpu(cp + 3, ew); }
      } else {
        cv.x = __fadd_rn(cv.x, ex); cv.y = __fadd_rn(cv.y, ey);
        cv.z = __fadd_rn(cv.z, ez); cv.w = __fadd_rn(cv.w, ew);
        __stcg(reinterpret_cast<float4*>(c + v * 4), cv);
      }
    }
    for (int64_t i = nv * 4 + tid; i < len; i += stride) {  // segment tail (last segment only)
      const float xi = xs[i];
      const float ci = __ldcg(c + i);
      const float e = elastic_diff(xi, ci, alpha);
      xs[i] = __fsub_rn(xi, e);
      if (Concurrent) { if (SYS) red_add_sys(c + i, e); else red_add_gpu(c + i, e); }
      else c[i] = __fadd_rn(ci, e);
    }
  }
}

// A whole server round in arrival order, fused: the centre is read once and
// written once; worker w's update uses the centre left by the previous one.
// Bitwise equal to serial updates in `order` (each element is independent).
constexpr int kMaxRoundWorkers = 16;
constexpr int kMaxRoundOrder = 64;
struct RoundArgs {
  float* w[kMaxRoundWorkers];
  int8_t order[kMaxRoundOrder];
  int norder;
};

__global__ void __launch_bounds__(kThreads)
easgd_round_kernel(const __grid_constant__ RoundArgs ra, float* c, int64_t n, float alpha,
                   int vec) {
  const int64_t stride = (int64_t)gridDim.x * kThreads;
  const int64_t tid = (int64_t)blockIdx.x * kThreads + threadIdx.x;
  int64_t done = 0;
  if (vec) {
    const int64_t nv = n / 4;
    for (int64_t v = tid; v < nv; v += stride) {
      float4 cv = ld16_f(c + v * 4);
      for (int t = 0; t < ra.norder; ++t) {
        float* wp = ra.w[ra.order[t]] + v * 4;
        float4 xv = *reinterpret_cast<const float4*>(wp);
        const float ex = elastic_diff(xv.x, cv.x, alpha), ey = elastic_diff(xv.y, cv.y, alpha);
        const float ez = elastic_diff(xv.z, cv.z, alpha), ew = elastic_diff(xv.w, cv.w, alpha);
        xv.x = __fsub_rn(xv.x, ex); xv.y = __fsub_rn(xv.y, ey);
        xv.z = __fsub_rn(xv.z, ez); xv.w = __fsub_rn(xv.w, ew);
        cv.x = __fadd_rn(cv.x, ex); cv.y = __fadd_rn(cv.y, ey);
        cv.z = __fadd_rn(cv.z, ez); cv.w = __fadd_rn(cv.w, ew);
        *reinterpret_cast<float4*>(wp) = xv;
      }
      st16_f(c + v * 4, cv);
    }
    done = nv * 4;
  }
  for (int64_t i = done + tid; i < n; i += stride) {
    float ci = c[i];
    for (int t = 0; t < ra.norder; ++t) {
      float* wp = ra.w[ra.order[t]] + i;
      const float xi = *wp;
      const float e = elastic_diff(xi, ci, alpha);
      *wp = __fsub_rn(xi, e);
      ci = __fadd_rn(ci, e);
    }
    c[i] = ci;
  }
}

// Arrival order with N DISTINCT workers (the common round: each worker once):
// all N worker loads are issued before the dependent chain of centre updates,
// so N + 1 independent 16-byte loads are in flight per thread.  `wo` holds the
// workers' pointers already in arrival order.
struct OrderedWorkers {
  float* wo[8];
};

template <int N>
__global__ void __launch_bounds__(kThreads)
easgd_round_distinct_kernel(const __grid_constant__ OrderedWorkers ow, float* c, int64_t n,
                            float alpha) {
  const int64_t stride = (int64_t)gridDim.x * kThreads;
  const int64_t tid = (int64_t)blockIdx.x * kThreads + threadIdx.x;
  const int64_t nv = n / 4;
  for (int64_t v = tid; v < nv; v += stride) {
    float4 cv = ld16_f(c + v * 4);
    float4 xv[N];
#pragma unroll
    for (int t = 0; t < N; ++t) xv[t] = ld16_f(ow.wo[t] + v * 4);
#pragma unroll
    for (int t = 0; t < N; ++t) {
      const float ex = elastic_diff(xv[t].x, cv.x, alpha), ey = elastic_diff(xv[t].y, cv.y, alpha);
      const float ez = elastic_diff(xv[t].z, cv.z, alpha), ew = elastic_diff(xv[t].w, cv.w, alpha);
      xv[t].x = __fsub_rn(xv[t].x, ex); xv[t].y = __fsub_rn(xv[t].y, ey);
      xv[t].z = __fsub_rn(xv[t].z, ez); xv[t].w = __fsub_rn(xv[t].w, ew);
      cv.x = __fadd_rn(cv.x, ex); cv.y = __fadd_rn(cv.y, ey);
      cv.z = __fadd_rn(cv.z, ez); cv.w = __fadd_rn(cv.w, ew);
      st16_f(ow.wo[t] + v * 4, xv[t]);
    }
    st16_f(c + v * 4, cv);
  }
  for (int64_t i = nv * 4 + tid; i < n; i += stride) {  // tail, scalar
    float ci = c[i];
#pragma unroll
    for (int t = 0; t < N; ++t) {
      const float xi = ow.wo[t][i];
      const float e = elastic_diff(xi, ci, alpha);
      ow.wo[t][i] = __fsub_rn(xi, e);
      ci = __fadd_rn(ci, e);
    }
    c[i] = ci;
  }
}

__global__ void __launch_bounds__(kThreads)
cast_rn16_kernel(const float* __restrict__ in, uint16_t* __restrict__ out, int64_t n) {
  const int64_t stride = (int64_t)gridDim.x * kThreads;
  for (int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x; i < n; i += stride) {
    const __half h = __float2half_rn(in[i]);  // cvt.rn.f16.f32, as in the exchange
    out[i] = *reinterpret_cast<const uint16_t*>(&h);
  }
}

template <int K, bool W16>
const void* exchange_fn(bool sys) {
  return sys ? reinterpret_cast<const void*>(&tm_exchange_kernel<K, W16, true>)
             : reinterpret_cast<const void*>(&tm_exchange_kernel<K, W16, false>);
}

const void* pick_exchange(int k, bool w16, bool sys) {
  switch (k) {
    case 2: return w16 ? exchange_fn<2, true>(sys) : exchange_fn<2, false>(sys);
    case 3: return w16 ? exchange_fn<3, true>(sys) : exchange_fn<3, false>(sys);
    case 4: return w16 ? exchange_fn<4, true>(sys) : exchange_fn<4, false>(sys);
    case 5: return w16 ? exchange_fn<5, true>(sys) : exchange_fn<5, false>(sys);
    case 6: return w16 ? exchange_fn<6, true>(sys) : exchange_fn<6, false>(sys);
    case 7: return w16 ? exchange_fn<7, true>(sys) : exchange_fn<7, false>(sys);
    case 8: return w16 ? exchange_fn<8, true>(sys) : exchange_fn<8, false>(sys);
    default: return nullptr;
  }
}

int sm_count(int device) {
  int n = 0;
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device);
  return n > 0 ? n : 1;
}

}  // namespace

int exchange_max_ctas(int device, bool wire16, int k) {
  const void* fn = pick_exchange(k, wire16, true);
  if (!fn) return 0;
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kThreads, 0) != cudaSuccess)
    return 0;
  return per_sm * sm_count(device);
}

int grid_for_streaming(int device) { return 4 * sm_count(device); }

cudaError_t launch_exchange(const ExchangeArgs& a, int nlocal, bool wire16, cudaStream_t s) {
  // System-scope flags only when some peer rank lives in another process
  // (another GPU, over NVLink); a single-process group syncs at GPU scope.
  const void* fn = pick_exchange(a.k, wire16, nlocal != a.k);
  if (!fn) return cudaErrorInvalidValue;
  void* params[] = {const_cast<ExchangeArgs*>(&a)};
  // Cooperative launch: guarantees every CTA is co-resident, which the
  // per-CTA flag barriers need when several ranks share this device.
  return cudaLaunchCooperativeKernel(fn, dim3(nlocal * a.C), dim3(kThreads), params, 0, s);
}

template <int K, bool Q16, int TILE, int RING_KB, int MINB>
cudaError_t launch_tma(const LocalBufs& lb, int64_t P, uint32_t* status, int dev, cudaStream_t s) {
  using Cfg = TmaCfg<K, TILE, RING_KB, MINB>;
  const int64_t ntiles = P / TILE;
  auto fn = tm_direct_tma_kernel<K, Q16, TILE, RING_KB, MINB>;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::kSmem);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  const int grid = (int)std::min<int64_t>(ntiles, (int64_t)MINB * sm_count(dev));
  fn<<<grid, kThreads, Cfg::kSmem, s>>>(lb, ntiles, P, status);
  return cudaGetLastError();
}

// Tuning knob (diagnostics only): TM_TMA_CFG selects the tile / ring / residency
// of the bulk-async kernel for k = 8; TM_DIRECT_LDG=1 forces the register path.
int env_int(const char* name, int dflt) {
  const char* v = getenv(name);
  return (v && *v) ? atoi(v) : dflt;
}

template <int K, bool Q16>
cudaError_t direct_tma(const LocalBufs& lb, int64_t P, uint32_t* status, int dev, cudaStream_t s) {
  if constexpr (K == 8) {
    static const int cfg = env_int("TM_TMA_CFG", 0);
    switch (cfg) {
      case 8: return launch_tma<K, Q16, 1024, 160, 1>(lb, P, status, dev, s);
      case 1: return launch_tma<K, Q16, 1024, 96, 2>(lb, P, status, dev, s);
      case 2: return launch_tma<K, Q16, 2048, 192, 1>(lb, P, status, dev, s);
      case 3: return launch_tma<K, Q16, 1024, 64, 2>(lb, P, status, dev, s);
      case 4: return launch_tma<K, Q16, 2048, 96, 2>(lb, P, status, dev, s);
      case 5: return launch_tma<K, Q16, 2048, 96, 1>(lb, P, status, dev, s);
      case 6: return launch_tma<K, Q16, 2048, 96, 3>(lb, P, status, dev, s);
      case 7: return launch_tma<K, Q16, 2048, 192, 1>(lb, P, status, dev, s);
      default: break;
    }
  }
  // Default, from the r01 sweep at k = 8 (profiles/r01/README.md): 8 KB tiles per
  // buffer, a 2-deep ring for k = 8 (128 KB in flight per SM), one CTA per SM.
  return launch_tma<K, Q16, 2048, 96, 1>(lb, P, status, dev, s);
}

template <int K>
cudaError_t direct_k(const LocalBufs& lb, int64_t P, uint32_t* status, bool q16, int dev,
                     cudaStream_t s) {
  static const bool force_ldg = env_int("TM_DIRECT_LDG", 0) == 1;
  if (P >= 2048 && !force_ldg)
    return q16 ? direct_tma<K, true>(lb, P, status, dev, s) : direct_tma<K, false>(lb, P, status, dev, s);
  const int64_t want = (P / 4 + kThreads - 1) / kThreads;
  const int per_sm = K >= 7 ? 3 : 4;  // = the kernel's __launch_bounds__ residency
  const int grid = (int)std::min<int64_t>(std::max<int64_t>(want, 1), per_sm * sm_count(dev));
  if (q16) tm_direct_kernel<K, true><<<grid, kThreads, 0, s>>>(lb, 0, P, status);
  else tm_direct_kernel<K, false><<<grid, kThreads, 0, s>>>(lb, 0, P, status);
  return cudaGetLastError();
}

cudaError_t launch_direct(float* const* bufs, int k, int64_t P, bool q16, uint32_t* status,
                          cudaStream_t s) {
  LocalBufs lb{};
  for (int j = 0; j < k; ++j) lb.b[j] = bufs[j];
  int dev = 0;
  cudaGetDevice(&dev);
  switch (k) {
    case 2: return direct_k<2>(lb, P, status, q16, dev, s);
    case 3: return direct_k<3>(lb, P, status, q16, dev, s);
    case 4: return direct_k<4>(lb, P, status, q16, dev, s);
    case 5: return direct_k<5>(lb, P, status, q16, dev, s);
    case 6: return direct_k<6>(lb, P, status, q16, dev, s);
    case 7: return direct_k<7>(lb, P, status, q16, dev, s);
    case 8: return direct_k<8>(lb, P, status, q16, dev, s);
    default: return cudaErrorInvalidValue;
  }
}

static int streaming_grid(int64_t work_items) {
  int dev = 0;
  cudaGetDevice(&dev);
  int64_t want = (work_items + kThreads - 1) / kThreads;
  return (int)std::min<int64_t>(std::max<int64_t>(want, 1), grid_for_streaming(dev));
}

cudaError_t launch_easgd(float* x, float* c, int64_t n, float alpha, bool concurrent,
                         cudaStream_t s) {
  const int vec = ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(c)) & 15) == 0;
  const int grid = streaming_grid(vec ? n / 4 + 4 : n);
  if (concurrent) easgd_kernel<true><<<grid, kThreads, 0, s>>>(x, c, n, alpha, vec);
  else easgd_kernel<false><<<grid, kThreads, 0, s>>>(x, c, n, alpha, vec);
  return cudaGetLastError();
}

cudaError_t launch_easgd_round(float* const* w, int nw, const int32_t* order, int norder,
                               float* c, int64_t n, float alpha, cudaStream_t s) {
  if (nw < 1 || nw > kMaxRoundWorkers || norder < 0 || norder > kMaxRoundOrder)
    return cudaErrorInvalidValue;
  RoundArgs ra{};
  uintptr_t align = reinterpret_cast<uintptr_t>(c);
  for (int i = 0; i < nw; ++i) {
    ra.w[i] = w[i];
    align |= reinterpret_cast<uintptr_t>(w[i]);
  }
  for (int t = 0; t < norder; ++t) {
    if (order[t] < 0 || order[t] >= nw) return cudaErrorInvalidValue;
    ra.order[t] = (int8_t)order[t];
  }
  ra.norder = norder;
  const int vec = (align & 15) == 0;
  bool distinct = norder >= 1 && norder <= 8;
  for (int t = 0; distinct && t < norder; ++t)
    for (int u = 0; u < t; ++u)
      if (order[u] == order[t]) distinct = false;
  if (vec && distinct) {
    OrderedWorkers ow{};
    for (int t = 0; t < norder; ++t) ow.wo[t] = w[order[t]];
    const int grid = streaming_grid(n / 4 + 4);
    switch (norder) {
#define TM_RD(N) \
  case N: easgd_round_distinct_kernel<N><<<grid, kThreads, 0, s>>>(ow, c, n, alpha); break;
      TM_RD(1) TM_RD(2) TM_RD(3) TM_RD(4) TM_RD(5) TM_RD(6) TM_RD(7) TM_RD(8)
#undef TM_RD
    }
    return cudaGetLastError();
  }
  const int grid = streaming_grid(vec ? n / 4 + 4 : n);
  easgd_round_kernel<<<grid, kThreads, 0, s>>>(ra, c, n, alpha, vec);
  return cudaGetLastError();
}

cudaError_t launch_easgd_sharded(float* x, const ShardArgs& sa, float alpha, bool concurrent,
                                 cudaStream_t s) {
  const int grid = streaming_grid(sa.L / 4 + 4);
  if (concurrent) {
    if (sa.sys) easgd_sharded_kernel<true, true><<<grid, kThreads, 0, s>>>(x, sa, alpha);
    else easgd_sharded_kernel<true, false><<<grid, kThreads, 0, s>>>(x, sa, alpha);
  } else {
    easgd_sharded_kernel<false, false><<<grid, kThreads, 0, s>>>(x, sa, alpha);
  }
  return cudaGetLastError();
}

cudaError_t launch_cast_rn16(const float* in, uint16_t* out, int64_t n, cudaStream_t s) {
  cast_rn16_kernel<<<streaming_grid(n), kThreads, 0, s>>>(in, out, n);
  return cudaGetLastError();
}

}  // namespace tmx
