// sm_100a kernels of the single-process ("direct") exchange path: all k ranks'
// buffers on one device, one pass, no staging and no flags (include/tm.h,
// TM_PATH_DIRECT).  PAPER L237-269 (ASA / ASA16), L233-237 (AR).
#include <cuda_fp16.h>
#include <stdint.h>
#include <stdlib.h>

#include <algorithm>

#include "tm_device.cuh"
#include "tm_internal.h"

namespace tmx {
namespace {
using namespace dev;

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
  int sum;     // SUBGD sum mode: no 1/k
  int l2hint;  // A/B knob TM_L2_HINT: bit 0 evict_first on the bulk loads, bit 1 on the bulk stores
};

// The method's arithmetic on 4 elements of k contributions (registers in, one
// float4 out): rn16 of each contribution (Q16), ascending-rank sum from the
// rank-0 term, fl(s/k), rn16 of the average.  `st` accumulates status bits.
template <int K, bool Q16>
__device__ __forceinline__ float4 average4(const float4 (&in)[K], uint32_t& st, bool sum) {
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
  if (!sum) {
    s.x = div_k<K>(s.x); s.y = div_k<K>(s.y); s.z = div_k<K>(s.z); s.w = div_k<K>(s.w);
  } else if (Q16) {  // a sum (unlike an average) can leave the binary16 range
    st |= (status_of(s.x, true) | status_of(s.y, true) | status_of(s.z, true) | status_of(s.w, true)) &
          TM_BIT_OVERFLOW16;
  }
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
  if (!lb.sum) s = div_k<K>(s);
  else if (Q16) st |= status_of(s, true) & TM_BIT_OVERFLOW16;
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
    const float4 s = average4<K, Q16>(in, st, lb.sum != 0);
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

template <int K, bool Q16, int TILE, int RING_KB, int MINB>
__global__ void __launch_bounds__(kThreads, MINB)
tm_direct_tma_kernel(const __grid_constant__ LocalBufs lb, int64_t ntiles, int64_t P,
                     uint32_t* status, unsigned long long* tile_ctr) {
  using Cfg = TmaCfg<K, TILE, RING_KB, MINB>;
  constexpr int S = Cfg::kStages;
  constexpr int V = Cfg::kVecPerThread;
  constexpr uint32_t TB = Cfg::kTileBytes;
  extern __shared__ __align__(128) unsigned char smem[];
  float* ring = reinterpret_cast<float*>(smem);                  // [S][K][TILE]
  float* outr = ring + (size_t)S * K * TILE;                     // [kOutRing][TILE]
  __shared__ __align__(16) uint64_t full[kMaxStages];
  __shared__ int64_t slot_tile[kMaxStages];  // tile held by each ring slot, -1 = none left
  static_assert(S <= kMaxStages, "ring depth");

  const int tid = threadIdx.x;
  const uint64_t pol = lb.l2hint ? l2_policy_evict_first() : 0;
  // Tiles are claimed dynamically from a per-launch counter (work stealing), so
  // a slow SM does not hold back the end of the kernel; without a counter the
  // static assignment blockIdx.x + i * gridDim.x is used.
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
  auto issue = [&](int64_t i) {  // thread 0: fill ring slot i % S with the next tile
    const int s = (int)(i % S);
    const int64_t t = claim();
    slot_tile[s] = t;  // published to the consumers by the mbarrier arrive below
    if (t < 0) {
      mbar_expect_tx(&full[s], 0);
      return;
    }
    mbar_expect_tx(&full[s], K * TB);
    if (lb.l2hint & 1) {
#pragma unroll
      for (int j = 0; j < K; ++j)
        bulk_load_hint(ring + ((size_t)s * K + j) * TILE, lb.b[j] + t * TILE, TB, &full[s], pol);
    } else {
#pragma unroll
      for (int j = 0; j < K; ++j)
        bulk_load(ring + ((size_t)s * K + j) * TILE, lb.b[j] + t * TILE, TB, &full[s]);
    }
  };

  if (tid == 0) {
    for (int s = 0; s < S; ++s) mbar_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int64_t i = 0; i < S; ++i) issue(i);
  }
  __syncthreads();

  uint32_t st = 0;
  for (int64_t i = 0;; ++i) {
    const int s = (int)(i % S);
    mbar_wait(&full[s], (uint32_t)((i / S) & 1));
    const int64_t t = slot_tile[s];
    if (t < 0) break;  // uniform: every later claim is past the end too
    float* out = outr + (size_t)(i % kOutRing) * TILE;
#pragma unroll
    for (int u = 0; u < V; ++u) {
      float4 in[K];
#pragma unroll
      for (int j = 0; j < K; ++j)
        in[j] = reinterpret_cast<const float4*>(ring + ((size_t)s * K + j) * TILE)[tid + u * kThreads];
      reinterpret_cast<float4*>(out)[tid + u * kThreads] = average4<K, Q16>(in, st, lb.sum != 0);
    }
    fence_proxy_async_smem();  // generic-proxy smem writes -> visible to the bulk store
    if (tid == 0) bulk_wait_read<kOutRing - 2>();  // out slot of tile i+1 is free
    __syncthreads();
    if (tid == 0) {
      if (lb.l2hint & 2) {
#pragma unroll
        for (int j = 0; j < K; ++j) bulk_store_hint(lb.b[j] + t * TILE, out, TB, pol);
      } else {
#pragma unroll
        for (int j = 0; j < K; ++j) bulk_store(lb.b[j] + t * TILE, out, TB);
      }
      bulk_commit();
      issue(i + S);  // every thread has finished reading ring slot s
    }
  }
  if (tid == 0) {
    if (tile_ctr) tile_ctr_retire(tile_ctr);
    bulk_wait_all<0>();
  }

  // elements past the last whole tile: register path (one CTA)
  if (blockIdx.x == gridDim.x - 1) {
    const int64_t e0 = ntiles * TILE;
    for (int64_t v = e0 / 4 + tid; v < P / 4; v += kThreads) {
      float4 in[K];
#pragma unroll
      for (int j = 0; j < K; ++j) in[j] = ld16_f(lb.b[j] + v * 4);
      const float4 r = average4<K, Q16>(in, st, lb.sum != 0);
#pragma unroll
      for (int j = 0; j < K; ++j) st16_f(lb.b[j] + v * 4, r);
    }
    const int64_t i = (P / 4) * 4 + tid;
    if (i < P) average1<K, Q16>(lb, i, st);
  }
  if (st) atomicOr(status, st);
}

}  // namespace

template <int K, bool Q16, int TILE, int RING_KB, int MINB>
cudaError_t launch_tma(const LocalBufs& lb, int64_t P, uint32_t* status, unsigned long long* ctr,
                       int dev, cudaStream_t s, int max_grid) {
  using Cfg = TmaCfg<K, TILE, RING_KB, MINB>;
  const int64_t ntiles = P / TILE;
  if (ntiles == 0) {  // smaller than one tile: the register kernel
    tm_direct_kernel<K, Q16><<<(int)std::max<int64_t>(1, (P / 4 + kThreads - 1) / kThreads), kThreads, 0, s>>>(
        lb, 0, P, status);
    return cudaGetLastError();
  }
  auto fn = tm_direct_tma_kernel<K, Q16, TILE, RING_KB, MINB>;
  static std::atomic<uint64_t> optin{0};
  cudaError_t e0 = smem_optin(reinterpret_cast<const void*>(fn), Cfg::kSmem, dev, optin);
  if (e0 != cudaSuccess) return e0;
  int64_t cap = (int64_t)MINB * sm_count(dev);
  if (max_grid > 0) cap = std::min<int64_t>(cap, max_grid);  // CTA budget of a bucket
  const int grid = (int)std::min<int64_t>(ntiles, cap);
  fn<<<grid, kThreads, Cfg::kSmem, s>>>(lb, ntiles, P, status, ctr);
  return cudaGetLastError();
}

// Tuning knobs (diagnostics only): TM_TMA_CFG selects the tile / ring / residency
// of the bulk-async kernel for k = 8; TM_DIRECT_LDG=1 forces the register path.
template <int K, bool Q16>
cudaError_t direct_tma(const LocalBufs& lb, int64_t P, uint32_t* status, unsigned long long* ctr,
                       int dev, cudaStream_t s, int max_grid) {
  if constexpr (K == 8) {
    static const int cfg = env_int("TM_TMA_CFG", 0);
    switch (cfg) {
      case 8: return launch_tma<K, Q16, 1024, 160, 1>(lb, P, status, ctr, dev, s, max_grid);
      case 1: return launch_tma<K, Q16, 1024, 96, 2>(lb, P, status, ctr, dev, s, max_grid);
      case 2: return launch_tma<K, Q16, 2048, 192, 1>(lb, P, status, ctr, dev, s, max_grid);
      case 3: return launch_tma<K, Q16, 1024, 64, 2>(lb, P, status, ctr, dev, s, max_grid);
      case 4: return launch_tma<K, Q16, 2048, 96, 2>(lb, P, status, ctr, dev, s, max_grid);
      case 5: return launch_tma<K, Q16, 2048, 96, 1>(lb, P, status, ctr, dev, s, max_grid);
      case 6: return launch_tma<K, Q16, 2048, 96, 3>(lb, P, status, ctr, dev, s, max_grid);
      case 7: return launch_tma<K, Q16, 2048, 192, 1>(lb, P, status, ctr, dev, s, max_grid);
      default: break;
    }
  }
  if constexpr (K <= 4) {  // A/B for small k: larger tiles / deeper rings
    static const int cfg = env_int("TM_TMA_CFG", 0);
    switch (cfg) {
      case 9: return launch_tma<K, Q16, 4096, 128, 1>(lb, P, status, ctr, dev, s, max_grid);
      case 10: return launch_tma<K, Q16, 2048, 128, 1>(lb, P, status, ctr, dev, s, max_grid);
      case 11: return launch_tma<K, Q16, 4096, 96, 1>(lb, P, status, ctr, dev, s, max_grid);
      case 12: return launch_tma<K, Q16, 2048, 160, 1>(lb, P, status, ctr, dev, s, max_grid);
      default: break;
    }
  }
  // k = 2: 16 KB tiles per buffer, 3-deep ring: 0.146 vs 0.160 ms at AlexNet size
  // (profiles/r01/direct_small_k_cfg.txt; k = 4 measures the same either way).
  if constexpr (K == 2) return launch_tma<K, Q16, 4096, 96, 1>(lb, P, status, ctr, dev, s, max_grid);
  // Default, from the r01 sweep at k = 8 (profiles/r01/README.md): 8 KB tiles per
  // buffer, a 2-deep ring for k = 8 (128 KB in flight per SM), one CTA per SM.
  // (With dynamic tiles every TM_TMA_CFG measures 0.570-0.572 ms; register stores
  // in place of the bulk stores measured 0.574 ms.)
  return launch_tma<K, Q16, 2048, 96, 1>(lb, P, status, ctr, dev, s, max_grid);
}

// Small exchanges are latency-bound: the register kernel spreads one float4 of
// every buffer per thread over many CTAs, while the TMA kernel walks 2048-element
// tiles one per CTA through a load -> compute -> store chain.  Measured with 64
// exchanges per CUDA graph (profiles/r02/latency/direct_{tma,ldg}.jsonl): k = 8
// 2.2 vs 4.7 us at P = 128 Ki, 4.3 vs 6.3 us at 512 Ki, 15.4 vs 14.4 us at 2 Mi;
// k = 4 at 2 Mi 7.2 vs 10.4 us.  So the register kernel up to k * P = 8 Mi
// elements (32 MB of fp32 inputs), the TMA kernel above.
constexpr int64_t kDirectLdgMaxElems = (int64_t)8 << 20;

template <int K>
cudaError_t direct_k(const LocalBufs& lb, int64_t P, uint32_t* status, unsigned long long* ctr,
                     bool q16, int dev, cudaStream_t s, int max_ctas) {
  static const bool force_ldg = env_int("TM_DIRECT_LDG", 0) == 1;
  static const bool force_tma = env_int("TM_DIRECT_TMA", 0) == 1;  // diagnostics: TMA at every size
  // A/B: budgeted buckets on the TMA kernel (read per budgeted call, so tests can switch it)
  const bool range_tma = max_ctas > 0 && env_int("TM_RANGE_TMA", 0) == 1;
  if (P >= 2048 && !force_ldg && (max_ctas <= 0 || range_tma) &&
      (force_tma || (int64_t)K * P > kDirectLdgMaxElems))
    return q16 ? direct_tma<K, true>(lb, P, status, ctr, dev, s, max_ctas)
               : direct_tma<K, false>(lb, P, status, ctr, dev, s, max_ctas);
  const int64_t want = (P / 4 + kThreads - 1) / kThreads;
  const int per_sm = K >= 7 ? 3 : 4;  // = the kernel's __launch_bounds__ residency
  const int64_t cap = max_ctas > 0 ? max_ctas : (int64_t)per_sm * sm_count(dev);
  const int grid = (int)std::min<int64_t>(std::max<int64_t>(want, 1), cap);
  if (q16) tm_direct_kernel<K, true><<<grid, kThreads, 0, s>>>(lb, 0, P, status);
  else tm_direct_kernel<K, false><<<grid, kThreads, 0, s>>>(lb, 0, P, status);
  return cudaGetLastError();
}

cudaError_t launch_direct(float* const* bufs, int k, int64_t P, bool q16, bool sum,
                          uint32_t* status, unsigned long long* tile_ctr, cudaStream_t s, int max_ctas) {
  LocalBufs lb{};
  lb.sum = sum ? 1 : 0;
  static const int l2hint = env_int("TM_L2_HINT", 0) & 3;
  lb.l2hint = l2hint;
  for (int j = 0; j < k; ++j) lb.b[j] = bufs[j];
  int dev = 0;
  cudaGetDevice(&dev);
  switch (k) {
    case 2: return direct_k<2>(lb, P, status, tile_ctr, q16, dev, s, max_ctas);
    case 3: return direct_k<3>(lb, P, status, tile_ctr, q16, dev, s, max_ctas);
    case 4: return direct_k<4>(lb, P, status, tile_ctr, q16, dev, s, max_ctas);
    case 5: return direct_k<5>(lb, P, status, tile_ctr, q16, dev, s, max_ctas);
    case 6: return direct_k<6>(lb, P, status, tile_ctr, q16, dev, s, max_ctas);
    case 7: return direct_k<7>(lb, P, status, tile_ctr, q16, dev, s, max_ctas);
    case 8: return direct_k<8>(lb, P, status, tile_ctr, q16, dev, s, max_ctas);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace tmx
