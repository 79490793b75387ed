// sm_100a kernels of the EASGD elastic update (SPEC
// L475) and the fp16 rounding test hook.
#include <cuda_fp16.h>
#include <stdint.h>
#include <stdlib.h>

#include <algorithm>
#include <mutex>

#include "tm_device.cuh"
#include "tm_internal.h"

namespace tmx {
namespace {
using namespace dev;

// ---------------------------------------------------------------------------
// EASGD elastic update, one fp32 op per step:
//   d = fl(x - c); e = fl(alpha d); x' = fl(x - e); c' = fl(c + e).
// Concurrent modes let several workers (possibly on other GPUs, through an IPC
// mapping) update one centre at once without lost updates; each worker then
// read a possibly stale c:
//   Mode 1: c += e with red.relaxed.sys.global.add(.v4).f32 -- the hardware
//           float atomic, which flushes fp32-subnormal operands and results to
//           signed zero;
//   Mode 2: c += e with a compare-and-swap loop around __fadd_rn -- one exact
//           IEEE add per update with gradual underflow (reading Q6), at the cost
//           of a CAS round trip per element;
//   Mode 3: Mode 2's arithmetic on 16-byte vectors with ONE 128-bit CAS
//           (atom.cas.b128, ATOMG.E.CAS.128) per 4 elements, its first expected
//           value the c the update was computed from (no second read): each
//           element still gets one exact add applied atomically, so the result
//           is one of Mode 2's interleavings.  Launched only when the centre is
//           on the launching GPU (the host checks; peers' memory keeps Mode 2).
// ---------------------------------------------------------------------------
template <bool SYS>
__device__ __forceinline__ void cas_add(float* p, float v, unsigned int old) {
  unsigned int* a = reinterpret_cast<unsigned int*>(p);
  for (;;) {
    const unsigned int want = __float_as_uint(__fadd_rn(__uint_as_float(old), v));
    const unsigned int got = SYS ? atomicCAS_system(a, old, want) : atomicCAS(a, old, want);
    if (got == old) break;
    old = got;
  }
}

// 128-bit compare-and-swap; on return (lo, hi) hold the value found
__device__ __forceinline__ bool cas128(void* p, uint64_t& lo, uint64_t& hi, uint64_t nlo, uint64_t nhi) {
  uint64_t olo, ohi;
  asm volatile("{\n\t.reg .b128 cmp, val, old;\n\t"
               "mov.b128 cmp, {%2, %3};\n\t"
               "mov.b128 val, {%4, %5};\n\t"
               "atom.relaxed.sys.global.cas.b128 old, [%6], cmp, val;\n\t"
               "mov.b128 {%0, %1}, old;\n\t}"
               : "=l"(olo), "=l"(ohi)
               : "l"(lo), "l"(hi), "l"(nlo), "l"(nhi), "l"(p)
               : "memory");
  const bool ok = olo == lo && ohi == hi;
  lo = olo;
  hi = ohi;
  return ok;
}
__device__ __forceinline__ uint64_t pack2(float a, float b) {
  return (uint64_t)__float_as_uint(b) << 32 | __float_as_uint(a);
}
__device__ __forceinline__ float lo_f(uint64_t v) { return __uint_as_float((uint32_t)v); }
__device__ __forceinline__ float hi_f(uint64_t v) { return __uint_as_float((uint32_t)(v >> 32)); }

// c += e; cv = the centre value e was computed from (the CAS modes' first guess)
template <int Mode, bool SYS>
__device__ __forceinline__ void centre_add4(float* c, float4 e, float4 cv) {
  if constexpr (Mode == 1) {
    if (SYS) red_add4_sys(c, e);
    else red_add4_gpu(c, e);
  } else if constexpr (Mode == 3) {
    uint64_t lo = pack2(cv.x, cv.y), hi = pack2(cv.z, cv.w);
    for (;;) {
      const uint64_t nlo = pack2(__fadd_rn(lo_f(lo), e.x), __fadd_rn(hi_f(lo), e.y));
      const uint64_t nhi = pack2(__fadd_rn(lo_f(hi), e.z), __fadd_rn(hi_f(hi), e.w));
      if (cas128(c, lo, hi, nlo, nhi)) break;
    }
  } else {
    cas_add<SYS>(c, e.x, __float_as_uint(cv.x));
    cas_add<SYS>(c + 1, e.y, __float_as_uint(cv.y));
    cas_add<SYS>(c + 2, e.z, __float_as_uint(cv.z));
    cas_add<SYS>(c + 3, e.w, __float_as_uint(cv.w));
  }
}
template <int Mode, bool SYS>
__device__ __forceinline__ void centre_add1(float* c, float e, float cv) {
  if constexpr (Mode == 1) {
    if (SYS) red_add_sys(c, e);
    else red_add_gpu(c, e);
  } else {  // Modes 2 and 3 (scalar tail)
    cas_add<SYS>(c, e, __float_as_uint(cv));
  }
}

template <int Mode>
__global__ void __launch_bounds__(kThreads)
easgd_kernel(float* __restrict__ x, float* c, int64_t n, float alpha, int vec) {
  constexpr bool Concurrent = Mode != 0;
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
        centre_add4<Mode, true>(c + v * 4, make_float4(ex, ey, ez, ew), cv);
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
    if (Concurrent) centre_add1<Mode, true>(c + i, e, ci);
    else c[i] = __fadd_rn(ci, e);
  }
}

// Elastic update against a centre sharded by segment: element i
// of segment s = i / L lives at shard[s][i - s*L], local or on peer s over NVLink.
// Segments are multiples of 256 elements, so a 16-byte vector never straddles
// two shards.  Concurrent mode: c += e by red.add at system scope when the
// shard may be on another GPU.
template <int Mode, bool SYS>
__global__ void __launch_bounds__(kThreads)
easgd_sharded_kernel(float* __restrict__ x, const __grid_constant__ ShardArgs sa, float alpha) {
  constexpr bool Concurrent = Mode != 0;
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
        centre_add4<Mode, SYS>(c + v * 4, make_float4(ex, ey, ez, ew), cv);
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
      if (Concurrent) centre_add1<Mode, SYS>(c + i, e, ci);
      else c[i] = __fadd_rn(ci, e);
    }
  }
}

// Locked (atomic per-chunk) update against the sharded centre.  Work item =
// one chunk of kLockChunk elements of one shard.  Thread 0 takes the chunk's
// spin lock (atomicCAS, system scope when peers are other GPUs), fences, and
// takes a ticket (the arrival position, logged for tests); the CTA applies the
// exclusive elastic update to the chunk (centre read/written through L2, .cg);
// every thread fences its writes, the CTA syncs, thread 0 releases the lock.
// A chunk is thus updated by one worker at a time, in arrival order: bitwise
// the serial EASGD sequence of that chunk's arrival order.
template <bool SYS>
__device__ __forceinline__ uint32_t cas_u32(uint32_t* p, uint32_t cmp, uint32_t val) {
  if constexpr (SYS) return atomicCAS_system(p, cmp, val);
  else return atomicCAS(p, cmp, val);
}
template <bool SYS>
__device__ __forceinline__ void fence_scope() {
  if constexpr (SYS) __threadfence_system();
  else __threadfence();
}

template <bool SYS>
__global__ void __launch_bounds__(kThreads)
easgd_locked_kernel(float* __restrict__ x, const __grid_constant__ ShardArgs sa, float alpha) {
  __shared__ int s_go;
  const int64_t nch = (sa.L + kLockChunk - 1) / kLockChunk;  // chunks per shard
  const int64_t total = (int64_t)sa.k * nch;
  for (int64_t it = blockIdx.x; it < total; it += gridDim.x) {
    const int s = (int)(it / nch);
    const int64_t q = it - (int64_t)s * nch;
    const int64_t len_s = min(sa.L, sa.P - (int64_t)s * sa.L);
    const int64_t c0 = q * kLockChunk;
    if (c0 >= len_s) continue;  // uniform across the CTA
    const int64_t n = min(kLockChunk, len_s - c0);
    if (threadIdx.x == 0) {
      uint32_t* lock = sa.locks[s] + q;
      int go = 1;
      if (cas_u32<SYS>(lock, 0u, 1u) != 0u) {
        const uint64_t t0 = globaltimer();
        while (cas_u32<SYS>(lock, 0u, 1u) != 0u) {
          if (globaltimer() - t0 > sa.timeout_ns) {
            atomicOr(sa.status, TM_BIT_TIMEOUT);
            go = 0;
            break;
          }
          __nanosleep(64);
        }
      }
      if (go) {
        fence_scope<SYS>();  // acquire: the previous holder's centre writes
        // ticket: the arrival position (an atomic so no stale L1 line is read)
        const uint32_t t = SYS ? atomicAdd_system(sa.tickets[s] + q, 1u) : atomicAdd(sa.tickets[s] + q, 1u);
        // the log holds log_stride arrivals per chunk: later ones are not recorded
        // (TM_BIT_LOG_OVERFLOW) instead of spilling into the next chunk's slots
        if (sa.order_log) {
          if (t < (uint32_t)sa.log_stride)
            sa.order_log[((int64_t)s * nch + q) * sa.log_stride + t] = sa.worker_id;
          else
            atomicOr(sa.status, TM_BIT_LOG_OVERFLOW);
        }
      }
      s_go = go;
    }
    __syncthreads();
    if (!s_go) return;
    float* c = sa.shard[s] + c0;
    float* xs = x + (int64_t)s * sa.L + c0;
    for (int64_t v = threadIdx.x; v < n / 4; v += kThreads) {
      float4 xv = ld16_f(xs + v * 4);
      float4 cv = __ldcg(reinterpret_cast<const float4*>(c + v * 4));
      const float ex = elastic_diff(xv.x, cv.x, alpha), ey = elastic_diff(xv.y, cv.y, alpha);
      const float ez = elastic_diff(xv.z, cv.z, alpha), ew = elastic_diff(xv.w, cv.w, alpha);
      xv.x = __fsub_rn(xv.x, ex); xv.y = __fsub_rn(xv.y, ey);
      xv.z = __fsub_rn(xv.z, ez); xv.w = __fsub_rn(xv.w, ew);
      cv.x = __fadd_rn(cv.x, ex); cv.y = __fadd_rn(cv.y, ey);
      cv.z = __fadd_rn(cv.z, ez); cv.w = __fadd_rn(cv.w, ew);
      st16_f(xs + v * 4, xv);
      __stcg(reinterpret_cast<float4*>(c + v * 4), cv);
    }
    for (int64_t i = (n / 4) * 4 + threadIdx.x; i < n; i += kThreads) {
      const float xi = xs[i];
      const float ci = __ldcg(c + i);
      const float e = elastic_diff(xi, ci, alpha);
      xs[i] = __fsub_rn(xi, e);
      __stcg(c + i, __fadd_rn(ci, e));
    }
    fence_scope<SYS>();  // release: this thread's centre writes before the unlock
    __syncthreads();
    if (threadIdx.x == 0) {
      if (SYS) atomicExch_system(sa.locks[s] + q, 0u);
      else atomicExch(sa.locks[s] + q, 0u);
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

// One float4 of the round: the centre and the N workers' values are loaded
// first (N + 1 independent loads in flight), then the dependent chain.
template <int N>
__device__ __forceinline__ void round_chain(float4& cv, float4 (&xv)[N], float alpha) {
#pragma unroll
  for (int t = 0; t < N; ++t) {
    const float ex = elastic_diff(xv[t].x, cv.x, alpha), ey = elastic_diff(xv[t].y, cv.y, alpha);
    const float ez = elastic_diff(xv[t].z, cv.z, alpha), ew = elastic_diff(xv[t].w, cv.w, alpha);
    xv[t].x = __fsub_rn(xv[t].x, ex); xv[t].y = __fsub_rn(xv[t].y, ey);
    xv[t].z = __fsub_rn(xv[t].z, ez); xv[t].w = __fsub_rn(xv[t].w, ew);
    cv.x = __fadd_rn(cv.x, ex); cv.y = __fadd_rn(cv.y, ey);
    cv.z = __fadd_rn(cv.z, ez); cv.w = __fadd_rn(cv.w, ew);
  }
}

template <int N>
__device__ __forceinline__ void round_vec(const OrderedWorkers& ow, float* c, int64_t v, float alpha) {
  float4 cv = ld16_f(c + v * 4);
  float4 xv[N];
#pragma unroll
  for (int t = 0; t < N; ++t) xv[t] = ld16_f(ow.wo[t] + v * 4);
  round_chain<N>(cv, xv, alpha);
#pragma unroll
  for (int t = 0; t < N; ++t) st16_f(ow.wo[t] + v * 4, xv[t]);
  st16_f(c + v * 4, cv);
}

template <int N>
__device__ __forceinline__ void round_scalar(const OrderedWorkers& ow, float* c, int64_t i, float alpha) {
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

template <int N>
__global__ void __launch_bounds__(kThreads)
easgd_round_distinct_kernel(const __grid_constant__ OrderedWorkers ow, float* c, int64_t n,
                            float alpha) {
  const int64_t stride = (int64_t)gridDim.x * kThreads;
  const int64_t tid = (int64_t)blockIdx.x * kThreads + threadIdx.x;
  const int64_t nv = n / 4;
  for (int64_t v = tid; v < nv; v += stride) round_vec<N>(ow, c, v, alpha);
  for (int64_t i = nv * 4 + tid; i < n; i += stride) round_scalar<N>(ow, c, i, alpha);
}

// The same round on the TMA engine: persistent, one CTA per SM, tiles of
// kRoundTile elements assigned statically (blockIdx + i * gridDim).  Thread 0
// bulk-loads the centre tile and the N worker tiles into a ring slot; every
// thread runs the chain on one float4; the N + 1 result tiles go to an output
// slot and are bulk-stored.  72 B per element for N = 8, each byte once.
constexpr int kRoundTile = 4 * kThreads;  // one float4 per thread
// Ring depth: the largest power of two (<= 8) whose slots fit 216 KB beside the
// two output slots.  Non-power-of-two depths (3, 5, 7) ran correctly but every
// mbarrier wait was reported "missing init" by compute-sanitizer synccheck (with
// racecheck hazards following from it); power-of-two depths are clean.
template <int N>
struct RoundTma {
  static constexpr uint32_t kTB = kRoundTile * 4;
  static constexpr int kIn = (N + 1) * (int)kTB;
  static constexpr int kFit = (216 * 1024 - 2 * kIn) / kIn;
  static constexpr int kStages = kFit >= 8 ? 8 : kFit >= 4 ? 4 : 2;
  static constexpr int kOutSlots = 2;
  static constexpr int kSmem = kStages * kIn + kOutSlots * kIn;
};

template <int N>
__global__ void __launch_bounds__(kThreads, 1)
easgd_round_tma_kernel(const __grid_constant__ OrderedWorkers ow, float* c, int64_t ntiles, int64_t n,
                       float alpha, unsigned long long* tile_ctr) {
  using R = RoundTma<N>;
  constexpr int S = R::kStages;
  constexpr int T = kRoundTile;
  extern __shared__ __align__(128) unsigned char smem[];
  float* ring = reinterpret_cast<float*>(smem);            // [S][N + 1][T]: centre, workers
  float* outr = ring + (size_t)S * (N + 1) * T;             // [kOutSlots][N + 1][T]
  __shared__ __align__(8) uint64_t full[S];
  __shared__ int64_t slot_tile[S];
  const uint32_t fb = smem_u32(&full[0]);  // one address computation for every barrier op
  const int tid = threadIdx.x;
  // tiles claimed from a per-launch counter (work stealing; self-resetting), or
  // the static assignment blockIdx + i * gridDim without one
  int64_t next_static = blockIdx.x;
  auto claim = [&]() -> int64_t {
    int64_t t;
    if (tile_ctr) {
      t = (int64_t)atomicAdd(tile_ctr, 1ull);
    } else {
      t = next_static;
      next_static += gridDim.x;
    }
    return t < ntiles ? t : -1;
  };
  // thread 0 issues the N + 1 copies of a tile (measured 0.705 ms vs 0.711 ms with
  // one copy per lane of warp 0 at AlexNet size, N = 8; register stores in place
  // of the bulk stores: 0.710 vs 0.709 ms, no gain)
  auto issue = [&](int64_t i) {  // thread 0: claim a tile for ring use i
    const int s = (int)(i % S);
    const int64_t t = claim();
    slot_tile[s] = t;  // published to the consumers by the mbarrier arrive
    if (t < 0) {
      mbar_expect_tx_a(fb + 8 * s, 0);
      return;
    }
    mbar_expect_tx_a(fb + 8 * s, (N + 1) * R::kTB);
#pragma unroll
    for (int q = 0; q <= N; ++q)
      bulk_load_a(ring + ((size_t)s * (N + 1) + q) * T, (q == 0 ? c : ow.wo[q - 1]) + t * T, R::kTB,
                  fb + 8 * s);
  };
  if (tid == 0) {
    for (int s = 0; s < S; ++s) mbar_init_a(fb + 8 * s, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (tid == 0)
    for (int64_t i = 0; i < S; ++i) issue(i);
  for (int64_t i = 0;; ++i) {
    const int s = (int)(i % S);
    mbar_wait_a(fb + 8 * s, (uint32_t)((i / S) & 1));
    const int64_t t = slot_tile[s];
    if (t < 0) break;  // uniform: every later claim is past the end too
    const float* src = ring + (size_t)s * (N + 1) * T;
    float* out = outr + (size_t)(i % R::kOutSlots) * (N + 1) * T;
    float4 cv = reinterpret_cast<const float4*>(src)[tid];
    float4 xv[N];
#pragma unroll
    for (int w = 0; w < N; ++w) xv[w] = reinterpret_cast<const float4*>(src + (size_t)(1 + w) * T)[tid];
    round_chain<N>(cv, xv, alpha);
    reinterpret_cast<float4*>(out)[tid] = cv;
#pragma unroll
    for (int w = 0; w < N; ++w) reinterpret_cast<float4*>(out + (size_t)(1 + w) * T)[tid] = xv[w];
    fence_proxy_async_smem();
    if (tid == 0) bulk_wait_read<R::kOutSlots - 2>();  // out slot of tile i+1 is free
    __syncthreads();
    if (tid == 0) {
#pragma unroll
      for (int q = 0; q <= N; ++q) bulk_store((q == 0 ? c : ow.wo[q - 1]) + t * T, out + (size_t)q * T, R::kTB);
      bulk_commit();
      issue(i + S);
    }
  }
  if (tid == 0) {
    if (tile_ctr) tile_ctr_retire(tile_ctr);
    bulk_wait_all<0>();
  }
  if (blockIdx.x == gridDim.x - 1) {  // past the last whole tile: register path
    for (int64_t v = ntiles * T / 4 + tid; v < n / 4; v += kThreads) round_vec<N>(ow, c, v, alpha);
    for (int64_t i = (n / 4) * 4 + tid; i < n; i += kThreads) round_scalar<N>(ow, c, i, alpha);
  }
}

// Per-device ring of kCtrSlots claim / retire pairs for the round kernel's
// dynamic tiles (the round needs no exchanger context): allocated and zeroed on
// first use; each launch takes the next pair, so rounds running concurrently on
// different streams (e.g. two centres) never claim tiles from one counter; each
// launch's last CTA resets its pair.  Null if the allocation failed (static
// tiles then).
unsigned long long* round_tile_ctr(int dev, bool may_allocate, cudaStream_t stream) {
  static std::mutex mu;
  static unsigned long long* ring[64] = {};
  static uint32_t seq[64] = {};
  std::lock_guard<std::mutex> lk(mu);
  if (dev < 0 || dev >= 64) return nullptr;
  if (!ring[dev]) {
    if (!may_allocate) return nullptr;
    void* p = nullptr;
    const size_t bytes = (size_t)kCtrSlots * 2 * sizeof(unsigned long long);
    if (cudaMalloc(&p, bytes) != cudaSuccess) return nullptr;
    // zeroed, and waited for, before any round on any stream claims from it (a
    // legacy-stream cudaMemset would not order a non-blocking stream's round)
    if (cudaMemsetAsync(p, 0, bytes, stream) != cudaSuccess || cudaStreamSynchronize(stream) != cudaSuccess) {
      cudaFree(p);
      return nullptr;
    }
    ring[dev] = static_cast<unsigned long long*>(p);
  }
  return ring[dev] + 2 * (size_t)(seq[dev]++ % kCtrSlots);
}

template <int N>
cudaError_t launch_round_tma(const OrderedWorkers& ow, float* c, int64_t n, int64_t ntiles, float alpha,
                             cudaStream_t s) {
  using R = RoundTma<N>;
  int dev = 0;
  cudaGetDevice(&dev);
  auto fn = easgd_round_tma_kernel<N>;
  static std::atomic<uint64_t> optin{0};
  cudaError_t e = smem_optin(reinterpret_cast<const void*>(fn), R::kSmem, dev, optin);
  if (e != cudaSuccess) return e;
  const int grid = (int)std::min<int64_t>(ntiles, sm_count(dev));
  static const bool stat = env_int("TM_ROUND_STATIC", 0) == 1;  // A/B: static tile assignment
  // no allocation while the stream is being captured: static tiles then
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(s, &cap);
  // Dynamic claims only for N >= 4: one counter serves ~60 K tiles per AlexNet-size
  // round, and with few workers a tile is so little work that the claims on that
  // one address become the limit (N = 1: 238 vs 153 us per update, static wins).
  unsigned long long* ctr =
      (stat || N < 4) ? nullptr : round_tile_ctr(dev, cap == cudaStreamCaptureStatusNone, s);
  fn<<<grid, kThreads, R::kSmem, s>>>(ow, c, ntiles, n, alpha, ctr);
  return cudaGetLastError();
}

// Small rounds are latency-bound: the register kernel beats the tile pipeline
// up to n (N + 1) = 18 Mi elements (N = 8: 1.8 vs 4.9 us at n = 4 Ki, 15.0 vs
// 19.3 us at 2 Mi, 51.3 vs 47.7 us at 4 Mi; profiles/r02/latency/small_bsp_easgd_*.jsonl).
constexpr int64_t kRoundLdgMaxElems = (int64_t)18 << 20;

template <int N>
cudaError_t launch_round_distinct(const OrderedWorkers& ow, float* c, int64_t n, float alpha,
                                  cudaStream_t s) {
  static const bool force_ldg = env_int("TM_DIRECT_LDG", 0) == 1;  // diagnostics: register kernel
  static const bool force_tma = env_int("TM_DIRECT_TMA", 0) == 1;  // diagnostics: TMA at every size
  const int64_t ntiles = n / kRoundTile;
  if (ntiles > 0 && !force_ldg && (force_tma || n * (N + 1) > kRoundLdgMaxElems)) {
    return launch_round_tma<N>(ow, c, n, ntiles, alpha, s);
  }
  easgd_round_distinct_kernel<N><<<streaming_grid(n / 4 + 4), kThreads, 0, s>>>(ow, c, n, alpha);
  return cudaGetLastError();
}

__global__ void __launch_bounds__(kThreads)
cast_rn16_kernel(const float* __restrict__ in, uint16_t* __restrict__ out, int64_t n) {
  const int64_t stride = (int64_t)gridDim.x * kThreads;
  for (int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x; i < n; i += stride) {
    const __half h = __float2half_rn(in[i]);  // cvt.rn.f16.f32, as in the exchange
    out[i] = *reinterpret_cast<const uint16_t*>(&h);
  }
}

// The 128-bit CAS of Mode 3 only on memory of the launching GPU (peer memory
// behind an IPC mapping keeps the 32-bit CAS of Mode 2); TM_EASGD_CAS128=0 turns
// it off (A/B), =2 forces it on peer memory too (for tools/multigpu_eval.sh:
// 128-bit atomics over NVLink are untested on the one-GPU boxes).
bool cas128_ok(const void* p) {
  const int mode = env_int("TM_EASGD_CAS128", 1);  // read per launch (tests switch it)
  if (mode == 0) return false;
  if (mode == 2) return true;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return false;
  cudaPointerAttributes at{};
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeDevice && at.device == dev;
}

}  // namespace

cudaError_t launch_easgd(float* x, float* c, int64_t n, float alpha, int concurrent,
                         cudaStream_t s) {
  const int vec = ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(c)) & 15) == 0;
  const int grid = streaming_grid(vec ? n / 4 + 4 : n);
  if (concurrent == 2 && vec && cas128_ok(c)) easgd_kernel<3><<<grid, kThreads, 0, s>>>(x, c, n, alpha, vec);
  else if (concurrent == 2) easgd_kernel<2><<<grid, kThreads, 0, s>>>(x, c, n, alpha, vec);
  else if (concurrent) easgd_kernel<1><<<grid, kThreads, 0, s>>>(x, c, n, alpha, vec);
  else easgd_kernel<0><<<grid, kThreads, 0, s>>>(x, c, n, alpha, vec);
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
    switch (norder) {
      case 1: return launch_round_distinct<1>(ow, c, n, alpha, s);
      case 2: return launch_round_distinct<2>(ow, c, n, alpha, s);
      case 3: return launch_round_distinct<3>(ow, c, n, alpha, s);
      case 4: return launch_round_distinct<4>(ow, c, n, alpha, s);
      case 5: return launch_round_distinct<5>(ow, c, n, alpha, s);
      case 6: return launch_round_distinct<6>(ow, c, n, alpha, s);
      case 7: return launch_round_distinct<7>(ow, c, n, alpha, s);
      default: return launch_round_distinct<8>(ow, c, n, alpha, s);
    }
  }
  const int grid = streaming_grid(vec ? n / 4 + 4 : n);
  easgd_round_kernel<<<grid, kThreads, 0, s>>>(ra, c, n, alpha, vec);
  return cudaGetLastError();
}

cudaError_t launch_easgd_sharded(float* x, const ShardArgs& sa, float alpha, int concurrent,
                                 cudaStream_t s) {
  const int grid = streaming_grid(sa.L / 4 + 4);
  bool local = concurrent == 2;  // every shard on this GPU: the 128-bit CAS
  for (int j = 0; local && j < sa.k; ++j) local = cas128_ok(sa.shard[j]);
  if (local) {
    easgd_sharded_kernel<3, true><<<grid, kThreads, 0, s>>>(x, sa, alpha);
  } else if (concurrent == 2) {
    if (sa.sys) easgd_sharded_kernel<2, true><<<grid, kThreads, 0, s>>>(x, sa, alpha);
    else easgd_sharded_kernel<2, false><<<grid, kThreads, 0, s>>>(x, sa, alpha);
  } else if (concurrent) {
    if (sa.sys) easgd_sharded_kernel<1, true><<<grid, kThreads, 0, s>>>(x, sa, alpha);
    else easgd_sharded_kernel<1, false><<<grid, kThreads, 0, s>>>(x, sa, alpha);
  } else {
    easgd_sharded_kernel<0, false><<<grid, kThreads, 0, s>>>(x, sa, alpha);
  }
  return cudaGetLastError();
}

cudaError_t launch_easgd_locked(float* x, const ShardArgs& sa, float alpha, cudaStream_t s) {
  const int64_t nch = (sa.L + kLockChunk - 1) / kLockChunk;
  int dev = 0;
  cudaGetDevice(&dev);
  const int grid = (int)std::min<int64_t>(std::max<int64_t>(sa.k * nch, 1), 4 * sm_count(dev));
  if (sa.sys) easgd_locked_kernel<true><<<grid, kThreads, 0, s>>>(x, sa, alpha);
  else easgd_locked_kernel<false><<<grid, kThreads, 0, s>>>(x, sa, alpha);
  return cudaGetLastError();
}

cudaError_t launch_cast_rn16(const float* in, uint16_t* out, int64_t n, cudaStream_t s) {
  cast_rn16_kernel<<<streaming_grid(n), kThreads, 0, s>>>(in, out, n);
  return cudaGetLastError();
}

}  // namespace tmx
