// sm_100a kernels of one BSP iteration's update + combine:
// the momentum-SGD step of every worker followed by
// the exchange of the weights and, optionally, of the velocities (PAPER
// L160-164, L373-376).
//
//   tm_bsp_tma_kernel     single-process group: ONE pass on the TMA engine.
//                         Persistent, one CTA per SM; thread 0 claims tiles of
//                         kTile elements from a per-launch counter and streams
//                         the k workers' (w, v, g) tiles into a shared-memory
//                         ring with cp.async.bulk; every thread takes the SGD
//                         step of 4 elements of every worker and averages the
//                         new weights (and velocities) with the exchange's
//                         arithmetic (rn16 of each contribution for ASA16,
//                         rank-order sum, fl(s/k), rn16) and stores the average
//                         into all k workers (and each worker's own v' when the
//                         velocities are not exchanged) from registers:
//                         12 B read + 8 B written per element per worker,
//                         instead of 20 B for the step plus 8 B (16 B with
//                         momentum) for a separate exchange.
//   tm_bsp_direct_kernel  the same arithmetic with 16-byte register loads
//                         (P smaller than one tile, TM_DIRECT_LDG=1); the TMA
//                         kernel's last CTA uses the same path for its tail.
//   sgd_kernel            the step alone (AR across processes, k = 1, and the
//                         TM_BSP_UNFUSED diagnostic).  On the staged path the
//                         step is fused into the exchange kernel's pre-cast
//                         (tm_staged.cu, ExchangeArgs::sgd): 12 B read + 6 B
//                         written (ASA16) per element instead of 20 B + 6 B.
// Every fp32 operation is one IEEE rounding: v' = fl(fl(mu v) - fl(lr g)),
// w' = fl(w + v').

#include <cuda_fp16.h>
#include <stdint.h>

#include <algorithm>

#include "tm_device.cuh"
#include "tm_internal.h"

namespace tmx {
namespace {
using namespace dev;

__device__ __forceinline__ uint32_t absmax4(float4 a) {
  return max(max(__float_as_uint(a.x) & 0x7fffffffu, __float_as_uint(a.y) & 0x7fffffffu),
             max(__float_as_uint(a.z) & 0x7fffffffu, __float_as_uint(a.w) & 0x7fffffffu));
}
__device__ __forceinline__ uint32_t status4(float4 a, bool q16) {
  return status_of(a.x, q16) | status_of(a.y, q16) | status_of(a.z, q16) | status_of(a.w, q16);
}
template <int K>
__device__ __forceinline__ float4 div4(float4 s) {
  return make_float4(div_k<K>(s.x), div_k<K>(s.y), div_k<K>(s.z), div_k<K>(s.w));
}
__device__ __forceinline__ float q1(float x) { return __half2float(__float2half_rn(x)); }

// The iteration's arithmetic on 4 elements of K workers: v[j] <- v'_j (the SGD
// step), sw <- average of the w'_j, sv <- average of the v'_j (MOM only).
template <int K, bool Q16, bool MOM>
__device__ __forceinline__ void bsp_core(const float4 (&w)[K], float4 (&v)[K], const float4 (&g)[K],
                                         float lr, float mu, float4& sw, float4& sv, uint32_t& st) {
  constexpr uint32_t thr = Q16 ? 0x477ff000u : 0x7f800000u;
#pragma unroll
  for (int j = 0; j < K; ++j) {
    const float4 vn = sgd_v(v[j], g[j], lr, mu);
    const float4 wn = add4(w[j], vn);
    v[j] = vn;
    uint32_t m = absmax4(wn);
    if (MOM) m = max(m, absmax4(vn));
    if (m >= thr) st |= status4(wn, Q16) | (MOM ? status4(vn, Q16) : 0u);
    const float4 tw = Q16 ? q16(wn) : wn;
    sw = j == 0 ? tw : add4(sw, tw);  // rank order from the rank-0 term
    if (MOM) {
      const float4 tv = Q16 ? q16(vn) : vn;
      sv = j == 0 ? tv : add4(sv, tv);
    }
  }
  sw = div4<K>(sw);
  if (Q16) sw = q16(sw);
  if (MOM) {
    sv = div4<K>(sv);
    if (Q16) sv = q16(sv);
  }
}

// One float4 (elements 4v .. 4v+3) through registers.
template <int K, bool Q16, bool MOM>
__device__ __forceinline__ void bsp_vec(const BspBufs& bb, int64_t v, uint32_t& st) {
  float4 w[K], vv[K], g[K];
#pragma unroll
  for (int j = 0; j < K; ++j) {
    w[j] = ld16_f(bb.w[j] + v * 4);
    vv[j] = ld16_f(bb.v[j] + v * 4);
    g[j] = ld16_f(bb.g[j] + v * 4);
  }
  float4 sw, sv;
  bsp_core<K, Q16, MOM>(w, vv, g, bb.lr, bb.mu, sw, sv, st);
#pragma unroll
  for (int j = 0; j < K; ++j) {
    st16_f(bb.w[j] + v * 4, sw);
    st16_f(bb.v[j] + v * 4, MOM ? sv : vv[j]);
  }
}

// One element (the last P % 4), scalar.
template <int K, bool Q16, bool MOM>
__device__ __forceinline__ void bsp_scalar(const BspBufs& bb, int64_t i, uint32_t& st) {
  float sw = 0.f, sv = 0.f;
#pragma unroll
  for (int j = 0; j < K; ++j) {
    const float vn = sgd_v1(bb.v[j][i], bb.g[j][i], bb.lr, bb.mu);
    const float wn = __fadd_rn(bb.w[j][i], vn);
    if (!MOM) bb.v[j][i] = vn;
    st |= status_of(wn, Q16) | (MOM ? status_of(vn, Q16) : 0u);
    const float tw = Q16 ? q1(wn) : wn;
    sw = j == 0 ? tw : __fadd_rn(sw, tw);
    if (MOM) {
      const float tv = Q16 ? q1(vn) : vn;
      sv = j == 0 ? tv : __fadd_rn(sv, tv);
    }
  }
  sw = div_k<K>(sw);
  if (Q16) sw = q1(sw);
#pragma unroll
  for (int j = 0; j < K; ++j) bb.w[j][i] = sw;
  if (MOM) {
    sv = div_k<K>(sv);
    if (Q16) sv = q1(sv);
#pragma unroll
    for (int j = 0; j < K; ++j) bb.v[j][i] = sv;
  }
}

// Register kernel over float4s [0, P/4) plus the scalar tail.
template <int K, bool Q16, bool MOM>
__global__ void __launch_bounds__(kThreads, 2)
tm_bsp_direct_kernel(const __grid_constant__ BspBufs bb, int64_t P, uint32_t* status) {
  const int64_t nv = P / 4;
  const int64_t stride = (int64_t)gridDim.x * kThreads;
  uint32_t st = 0;
  for (int64_t v = (int64_t)blockIdx.x * kThreads + threadIdx.x; v < nv; v += stride)
    bsp_vec<K, Q16, MOM>(bb, v, st);
  const int64_t i = nv * 4 + threadIdx.x;
  if (blockIdx.x == 0 && i < P) bsp_scalar<K, Q16, MOM>(bb, i, st);
  if (st) atomicOr(status, st);
}

// ---------------------------------------------------------------------------
// TMA-engine kernel.  Ring slot = the tile's 3K source tiles [w_0..w_{K-1} |
// v_0.. | g_0..]; output slot = [avg w | avg v (MOM) or v'_0..v'_{K-1}].
// ---------------------------------------------------------------------------
// Loads: thread 0 issues every bulk copy of a tile (measured faster than one
// copy per lane of warp 0: 1.65 vs 1.86-1.91 ms at AlexNet k = 8, 512-element tiles).  Stores: each
// thread writes its results with 16-byte register stores (128 threads x 16 B =
// one coalesced 2 KB row per buffer), measured 1.48 ms against 1.60 ms for bulk
// stores from an output ring (whose smem reads queue behind the ring's loads) and
// 1.57 ms for register stores with an "empty" mbarrier in place of __syncthreads.
template <int K, bool MOM, int TILE = 512>
struct BspTma {
  static constexpr int kTile = TILE;                  // elements per buffer per tile
  static constexpr int kThr = kTile / 4;              // one float4 per thread
  static constexpr uint32_t kTB = kTile * 4;          // bytes per buffer tile
  static constexpr int kInBytes = 3 * K * kTB;        // one ring slot
  static constexpr int kRaw = (200 * 1024) / kInBytes;
  static constexpr int kStages = kRaw > 8 ? 8 : (kRaw < 2 ? 2 : kRaw);
  static constexpr int kSmem = kStages * kInBytes;
};

template <int K, bool Q16, bool MOM, int TILE>
__global__ void __launch_bounds__(BspTma<K, MOM, TILE>::kThr, 1)
tm_bsp_tma_kernel(const __grid_constant__ BspBufs bb, int64_t ntiles, int64_t P, uint32_t* status,
                  unsigned long long* tile_ctr) {
  using C = BspTma<K, MOM, TILE>;
  constexpr int S = C::kStages;
  constexpr int T = C::kTile;
  extern __shared__ __align__(128) unsigned char smem[];
  float* ring = reinterpret_cast<float*>(smem);              // [S][3][K][T]
  __shared__ __align__(16) uint64_t full[kMaxStages];
  __shared__ int64_t slot_tile[kMaxStages];
  static_assert(S <= kMaxStages, "ring depth");
  const int tid = threadIdx.x;

  auto issue = [&](int64_t i) {  // thread 0: claim a tile for ring use i
    const int s = (int)(i % S);
    int64_t t = (int64_t)atomicAdd(tile_ctr, 1ull);
    if (t >= ntiles) t = -1;
    slot_tile[s] = t;  // published to the consumers by the mbarrier arrive
    if (t < 0) {
      mbar_expect_tx(&full[s], 0);
      return;
    }
    mbar_expect_tx(&full[s], 3 * K * C::kTB);
    float* dst = ring + (size_t)s * 3 * K * T;
#pragma unroll
    for (int j = 0; j < K; ++j) {
      bulk_load(dst + (size_t)j * T, bb.w[j] + t * T, C::kTB, &full[s]);
      bulk_load(dst + (size_t)(K + j) * T, bb.v[j] + t * T, C::kTB, &full[s]);
      bulk_load(dst + (size_t)(2 * K + j) * T, bb.g[j] + t * T, C::kTB, &full[s]);
    }
  };

  if (tid == 0) {
    for (int s = 0; s < S; ++s) mbar_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (tid == 0)
    for (int64_t i = 0; i < S; ++i) issue(i);

  uint32_t st = 0;
  for (int64_t i = 0;; ++i) {
    const int s = (int)(i % S);
    mbar_wait(&full[s], (uint32_t)((i / S) & 1));
    const int64_t t = slot_tile[s];
    if (t < 0) break;  // uniform: every later claim is past the end too
    const float* src = ring + (size_t)s * 3 * K * T;
    float4 w[K], v[K], g[K];
#pragma unroll
    for (int j = 0; j < K; ++j) {
      w[j] = reinterpret_cast<const float4*>(src + (size_t)j * T)[tid];
      v[j] = reinterpret_cast<const float4*>(src + (size_t)(K + j) * T)[tid];
      g[j] = reinterpret_cast<const float4*>(src + (size_t)(2 * K + j) * T)[tid];
    }
    float4 sw, sv;
    bsp_core<K, Q16, MOM>(w, v, g, bb.lr, bb.mu, sw, sv, st);
#pragma unroll
    for (int j = 0; j < K; ++j) {
      st16_f(bb.w[j] + t * T + tid * 4, sw);
      st16_f(bb.v[j] + t * T + tid * 4, MOM ? sv : v[j]);
    }
    __syncthreads();  // every thread is done with ring slot s
    if (tid == 0) issue(i + S);
  }
  if (tid == 0) tile_ctr_retire(tile_ctr);
  // elements past the last whole tile: register path (last CTA)
  if (blockIdx.x == gridDim.x - 1) {
    for (int64_t v = ntiles * T / 4 + tid; v < P / 4; v += C::kThr) bsp_vec<K, Q16, MOM>(bb, v, st);
    for (int64_t i = (P / 4) * 4 + tid; i < P; i += C::kThr) bsp_scalar<K, Q16, MOM>(bb, i, st);
  }
  if (st) atomicOr(status, st);
}

__global__ void __launch_bounds__(kThreads)
sgd_kernel(float* __restrict__ w, float* __restrict__ v, const float* __restrict__ g, int64_t n,
           float lr, float mu) {
  const int64_t stride = (int64_t)gridDim.x * kThreads;
  const int64_t tid = (int64_t)blockIdx.x * kThreads + threadIdx.x;
  const int64_t nv = n / 4;
  for (int64_t i = tid; i < nv; i += stride) {
    const float4 vn = sgd_v(ld16_f(v + i * 4), ld16_f(g + i * 4), lr, mu);
    st16_f(v + i * 4, vn);
    st16_f(w + i * 4, add4(ld16_f(w + i * 4), vn));
  }
  for (int64_t i = nv * 4 + tid; i < n; i += stride) {
    const float vn = sgd_v1(v[i], g[i], lr, mu);
    v[i] = vn;
    w[i] = __fadd_rn(w[i], vn);
  }
}

template <int K, bool Q16, bool MOM, int TILE>
cudaError_t bsp_tma_launch(const BspBufs& bb, int64_t P, uint32_t* status, unsigned long long* ctr,
                           int dev, cudaStream_t s) {
  using C = BspTma<K, MOM, TILE>;
  const int64_t ntiles = P / C::kTile;
  auto fn = tm_bsp_tma_kernel<K, Q16, MOM, TILE>;
  static std::atomic<uint64_t> optin{0};
  cudaError_t e = smem_optin(reinterpret_cast<const void*>(fn), C::kSmem, dev, optin);
  if (e != cudaSuccess) return e;
  const int grid = (int)std::min<int64_t>(ntiles, sm_count(dev));
  fn<<<grid, C::kThr, C::kSmem, s>>>(bb, ntiles, P, status, ctr);
  return cudaGetLastError();
}

// Small steps are latency-bound: the register kernel (one float4 of every
// buffer per thread, many CTAs) beats the tile pipeline up to k * P = 4 Mi
// elements (k = 8, momentum exchanged: 3.5 vs 5.6 us at P = 4 Ki, 9.5 vs 11.9 us
// at 512 Ki, 21.9 vs 21.0 us at 1 Mi; profiles/r02/latency/small_bsp_easgd_*.jsonl).
constexpr int64_t kBspLdgMaxElems = (int64_t)4 << 20;

template <int K, bool Q16, bool MOM>
cudaError_t bsp_launch(const BspBufs& bb, int64_t P, uint32_t* status, unsigned long long* ctr,
                       int dev, cudaStream_t s) {
  static const bool force_tma = env_int("TM_DIRECT_TMA", 0) == 1;  // diagnostics: TMA at every size
  if (ctr && (force_tma || (int64_t)K * P > kBspLdgMaxElems)) {
    // Tile per buffer: 2048 elements for k <= 4, 1024 above (AlexNet size: k = 2 / 4 /
    // 8 at 355 / 707 / 1421 us = 1.05 of the copy peak, vs 578 / 876 / 1478 us with
    // 512-element tiles, whose per-tile overhead dominated at small k;
    // profiles/r01/bsp_tile_ab.txt).  TM_BSP_TILE = 512 | 1024 | 2048 overrides.
    static const int tile = env_int("TM_BSP_TILE", K <= 4 ? 2048 : 1024);
    if constexpr (K <= 4)
      if (tile == 2048 && P >= 2048) return bsp_tma_launch<K, Q16, MOM, 2048>(bb, P, status, ctr, dev, s);
    if (tile == 1024 && P >= 1024) return bsp_tma_launch<K, Q16, MOM, 1024>(bb, P, status, ctr, dev, s);
    if (P >= 512) return bsp_tma_launch<K, Q16, MOM, 512>(bb, P, status, ctr, dev, s);
  }
  const int64_t want = (P / 4 + kThreads - 1) / kThreads;
  const int grid = (int)std::min<int64_t>(std::max<int64_t>(want, 1), 2 * sm_count(dev));
  tm_bsp_direct_kernel<K, Q16, MOM><<<grid, kThreads, 0, s>>>(bb, P, status);
  return cudaGetLastError();
}

template <int K>
cudaError_t bsp_k(const BspBufs& bb, int64_t P, bool q16, bool mom, uint32_t* status,
                  unsigned long long* ctr, int dev, cudaStream_t s) {
  if (q16) return mom ? bsp_launch<K, true, true>(bb, P, status, ctr, dev, s)
                      : bsp_launch<K, true, false>(bb, P, status, ctr, dev, s);
  return mom ? bsp_launch<K, false, true>(bb, P, status, ctr, dev, s)
             : bsp_launch<K, false, false>(bb, P, status, ctr, dev, s);
}

}  // namespace

cudaError_t launch_bsp_direct(const BspBufs& bb, int k, int64_t P, bool q16, bool mom,
                              uint32_t* status, unsigned long long* tile_ctr, cudaStream_t s) {
  int dev = 0;
  cudaGetDevice(&dev);
  static const bool force_ldg = env_int("TM_DIRECT_LDG", 0) == 1;  // diagnostics: register kernel
  unsigned long long* ctr = force_ldg ? nullptr : tile_ctr;
  switch (k) {
    case 2: return bsp_k<2>(bb, P, q16, mom, status, ctr, dev, s);
    case 3: return bsp_k<3>(bb, P, q16, mom, status, ctr, dev, s);
    case 4: return bsp_k<4>(bb, P, q16, mom, status, ctr, dev, s);
    case 5: return bsp_k<5>(bb, P, q16, mom, status, ctr, dev, s);
    case 6: return bsp_k<6>(bb, P, q16, mom, status, ctr, dev, s);
    case 7: return bsp_k<7>(bb, P, q16, mom, status, ctr, dev, s);
    case 8: return bsp_k<8>(bb, P, q16, mom, status, ctr, dev, s);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_sgd(float* w, float* v, const float* g, int64_t n, float lr, float mu,
                       cudaStream_t s) {
  sgd_kernel<<<streaming_grid(n / 4 + 4), kThreads, 0, s>>>(w, v, g, n, lr, mu);
  return cudaGetLastError();
}

}  // namespace tmx
