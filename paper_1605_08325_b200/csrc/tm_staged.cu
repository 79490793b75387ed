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

#include "tm_device.cuh"
#include "tm_internal.h"

namespace tmx {
namespace {
using namespace dev;

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

}  // namespace

int exchange_max_ctas(int device, bool wire16, int k) {
  const void* fn = pick_exchange(k, wire16, true);
  if (!fn) return 0;
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kThreads, 0) != cudaSuccess)
    return 0;
  return per_sm * sm_count(device);
}

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

}  // namespace tmx
