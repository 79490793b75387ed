// sm_100a kernels of one BSP iteration's update + combine:
// the momentum-SGD step of every worker followed by
// the exchange of the weights and, optionally, of the velocities (PAPER
// L160-164, L373-376).
//
//   tm_bsp_direct_kernel  single-process group: ONE pass.  For each element the
//                         k workers' (w, v, g) are read once, the SGD step is
//                         applied in registers, the new weights (and
//                         velocities) are averaged with the exchange's
//                         arithmetic (rn16 of each contribution for ASA16,
//                         rank-order sum, fl(s/k), rn16) and written to all k
//                         workers: 12 B read + 8 B written per element per
//                         worker, instead of 20 B for the step plus 8 B (16 B
//                         with momentum) for a separate exchange.
//   sgd_kernel            the step alone (multi-process path: step, then the
//                         staged exchange of w, and of v if requested).
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

__device__ __forceinline__ float4 sgd_v(float4 v, float4 g, float lr, float mu) {
  return make_float4(__fsub_rn(__fmul_rn(mu, v.x), __fmul_rn(lr, g.x)),
                     __fsub_rn(__fmul_rn(mu, v.y), __fmul_rn(lr, g.y)),
                     __fsub_rn(__fmul_rn(mu, v.z), __fmul_rn(lr, g.z)),
                     __fsub_rn(__fmul_rn(mu, v.w), __fmul_rn(lr, g.w)));
}
__device__ __forceinline__ float4 add4(float4 a, float4 b) {
  return make_float4(__fadd_rn(a.x, b.x), __fadd_rn(a.y, b.y), __fadd_rn(a.z, b.z), __fadd_rn(a.w, b.w));
}
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

template <int K, bool Q16, bool MOM>
__global__ void __launch_bounds__(kThreads, 2)
tm_bsp_direct_kernel(const __grid_constant__ BspBufs bb, int64_t P, uint32_t* status) {
  const int64_t nv = P / 4;
  const int64_t stride = (int64_t)gridDim.x * kThreads;
  const uint32_t thr = Q16 ? 0x477ff000u : 0x7f800000u;
  uint32_t st = 0;
  for (int64_t v = (int64_t)blockIdx.x * kThreads + threadIdx.x; v < nv; v += stride) {
    float4 sw = make_float4(0.f, 0.f, 0.f, 0.f), sv = sw;
#pragma unroll
    for (int j = 0; j < K; ++j) {
      const float4 w = ld16_f(bb.w[j] + v * 4);
      const float4 vv = ld16_f(bb.v[j] + v * 4);
      const float4 g = ld16_f(bb.g[j] + v * 4);
      const float4 vn = sgd_v(vv, g, bb.lr, bb.mu);
      const float4 wn = add4(w, vn);
      if (!MOM) st16_f(bb.v[j] + v * 4, vn);
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
#pragma unroll
    for (int j = 0; j < K; ++j) st16_f(bb.w[j] + v * 4, sw);
    if (MOM) {
      sv = div4<K>(sv);
      if (Q16) sv = q16(sv);
#pragma unroll
      for (int j = 0; j < K; ++j) st16_f(bb.v[j] + v * 4, sv);
    }
  }
  const int64_t i = nv * 4 + threadIdx.x;  // tail (P % 4 elements)
  if (blockIdx.x == 0 && i < P) {
    float sw = 0.f, sv = 0.f;
#pragma unroll
    for (int j = 0; j < K; ++j) {
      const float vn = __fsub_rn(__fmul_rn(bb.mu, bb.v[j][i]), __fmul_rn(bb.lr, bb.g[j][i]));
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
    const float vn = __fsub_rn(__fmul_rn(mu, v[i]), __fmul_rn(lr, g[i]));
    v[i] = vn;
    w[i] = __fadd_rn(w[i], vn);
  }
}

template <int K>
void bsp_k(const BspBufs& bb, int64_t P, bool q16, bool mom, uint32_t* status, int grid,
           cudaStream_t s) {
  if (q16) {
    if (mom) tm_bsp_direct_kernel<K, true, true><<<grid, kThreads, 0, s>>>(bb, P, status);
    else tm_bsp_direct_kernel<K, true, false><<<grid, kThreads, 0, s>>>(bb, P, status);
  } else {
    if (mom) tm_bsp_direct_kernel<K, false, true><<<grid, kThreads, 0, s>>>(bb, P, status);
    else tm_bsp_direct_kernel<K, false, false><<<grid, kThreads, 0, s>>>(bb, P, status);
  }
}

}  // namespace

cudaError_t launch_bsp_direct(const BspBufs& bb, int k, int64_t P, bool q16, bool mom,
                              uint32_t* status, cudaStream_t s) {
  int dev = 0;
  cudaGetDevice(&dev);
  const int64_t want = (P / 4 + kThreads - 1) / kThreads;
  const int grid = (int)std::min<int64_t>(std::max<int64_t>(want, 1), 2 * sm_count(dev));
  switch (k) {
    case 2: bsp_k<2>(bb, P, q16, mom, status, grid, s); break;
    case 3: bsp_k<3>(bb, P, q16, mom, status, grid, s); break;
    case 4: bsp_k<4>(bb, P, q16, mom, status, grid, s); break;
    case 5: bsp_k<5>(bb, P, q16, mom, status, grid, s); break;
    case 6: bsp_k<6>(bb, P, q16, mom, status, grid, s); break;
    case 7: bsp_k<7>(bb, P, q16, mom, status, grid, s); break;
    case 8: bsp_k<8>(bb, P, q16, mom, status, grid, s); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

cudaError_t launch_sgd(float* w, float* v, const float* g, int64_t n, float lr, float mu,
                       cudaStream_t s) {
  sgd_kernel<<<streaming_grid(n / 4 + 4), kThreads, 0, s>>>(w, v, g, n, lr, mu);
  return cudaGetLastError();
}

}  // namespace tmx
