// sm_100a kernels of the Theano-MPI parameter exchange (arXiv 1605.08325):
// the staged path, one persistent cooperative launch per exchange.  Kernel
// templates shared by tm_staged.cu (plain exchange) and tm_staged_sgd.cu (the
// exchange with the momentum-SGD step fused into its pre-cast, SGD = true): two
// translation units, so each kernel's register allocation is its own and the two
// sets compile in parallel.  Every definition is internal to the including
// translation unit.
//
// Five flavours (results bitwise identical; the runtime picks one at init by
// segment length and k):
//   tm_exchange_oneshot_kernel one barrier per call: every rank reduces every
//                             segment from every rank's staging (small segments);
//   tm_exchange_kernel        phases in sequence, 16-byte register loads/stores;
//   tm_exchange_ws_kernel     caster warps / reducer warps overlap a2 and a4 per
//                             sub-chunk, register loads;
//   tm_exchange_tma_kernel    phases in sequence as bulk-copy (TMA engine) tile
//                             pipelines (single-process default above the small sizes);
//   tm_exchange_tmaws_kernel  the ws overlap with TMA pipelines in both warp
//                             groups (multi-process default above the small sizes).
// Every flavour also exchanges a second vector between the same barriers
// (ExchangeArgs::nvec = 2: the BSP step with momentum exchange).
// The TMA phases (precast_phase / reduce_phase / gather_phase) are written once
// and parameterised by the thread group that runs them (Grp: whole CTA or half).
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

#pragma once

#include <cuda_fp16.h>
#include <stdint.h>
#include <stdlib.h>

#include <algorithm>

#include "tm_device.cuh"
#include "tm_internal.h"

namespace tmx {
namespace {
using namespace dev;

// Diagnostics: CTA-wide timestamp at a phase boundary (kernel-uniform branch;
// costs nothing when the log is off).
__device__ __forceinline__ void stamp(const ExchangeArgs& a, int slot) {
  if (a.stamps) {
    __syncthreads();
    if (threadIdx.x == 0) a.stamps[(size_t)blockIdx.x * kStampSlots + slot] = globaltimer();
  }
}

// Cross-rank, per-CTA epoch barrier (see the protocol in the file header).
// Returns false (whole CTA) if a peer timed out.
template <int K, bool SYS>
__device__ __forceinline__ bool rank_barrier(const ExchangeArgs& a, int phase, int r, int c,
                                             uint32_t epoch, int* s_abort) {
  __syncthreads();
  if (threadIdx.x < K) {
    const int j = threadIdx.x;
    uint32_t* remote = a.flags[j] + (size_t)(phase * TM_MAX_RANKS + r) * a.flag_stride + c;
    st_release<SYS>(remote, epoch);
    const uint32_t* mine = a.flags[r] + (size_t)(phase * TM_MAX_RANKS + j) * a.flag_stride + c;
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

// a2 for one wire unit (E elements at segment offset ev) of all K segments:
// load the fp32 source -- or, for the fused BSP step (a.sgd), compute it:
// v' = fl(fl(mu v) - fl(lr g)) is written back to v, the source is w' = fl(w + v')
// -- screen it and store its wire encoding into the own stage.  G segments per
// batch, all loads of a batch issued before any store (memory-level parallelism).
template <bool W16, int K, bool SGD>
__device__ __forceinline__ void precast_unit(const ExchangeArgs& a, int lr, int64_t ev,
                                             char* stage_r, uint32_t& st) {
  using U = Unit<W16>;
  constexpr int E = U::kElems;
  constexpr int WB = W16 ? 2 : 4;
  constexpr int G0 = SGD ? 1 : 4;  // SGD: 3 sources per unit; keep the register budget of the plain cast
  constexpr int G = K < G0 ? K : G0;
  const float* __restrict__ x = a.x[lr];
  const int64_t P = a.P, L = a.L;
#pragma unroll
  for (int s0 = 0; s0 < K; s0 += G) {
    float f[G][E];
    float fv[SGD ? G : 1][E], fg[SGD ? G : 1][E];
#pragma unroll
    for (int u = 0; u < G; ++u) {
      if (s0 + u < K) {
        const int64_t g = (int64_t)(s0 + u) * L + ev;
        if (g + E <= P) {
#pragma unroll
          for (int q = 0; q < E; q += 4) {
            const float4 t = ld16_f(x + g + q);
            f[u][q] = t.x; f[u][q + 1] = t.y; f[u][q + 2] = t.z; f[u][q + 3] = t.w;
            if constexpr (SGD) {
              const float4 tv = ld16_f(a.v[lr] + g + q), tg = ld16_f(a.g[lr] + g + q);
              fv[u][q] = tv.x; fv[u][q + 1] = tv.y; fv[u][q + 2] = tv.z; fv[u][q + 3] = tv.w;
              fg[u][q] = tg.x; fg[u][q + 1] = tg.y; fg[u][q + 2] = tg.z; fg[u][q + 3] = tg.w;
            }
          }
        } else {
#pragma unroll
          for (int q = 0; q < E; ++q) {
            const bool in = g + q < P;
            f[u][q] = in ? x[g + q] : 0.0f;
            if constexpr (SGD) {
              fv[u][q] = in ? a.v[lr][g + q] : 0.0f;
              fg[u][q] = in ? a.g[lr][g + q] : 0.0f;
            }
          }
        }
      }
    }
#pragma unroll
    for (int u = 0; u < G; ++u) {
      if (s0 + u < K) {
        const int64_t g = (int64_t)(s0 + u) * L + ev;
        if constexpr (SGD) {
#pragma unroll
          for (int q = 0; q < E; ++q) {
            fv[u][q] = g + q < P ? sgd_v1(fv[u][q], fg[u][q], a.lr, a.mu) : 0.0f;
            f[u][q] = g + q < P ? __fadd_rn(f[u][q], fv[u][q]) : 0.0f;
          }
          if (a.nvec == 2) {  // momentum exchanged: v' goes to the wire (vector 1), not back to v
            st |= unit_status<W16, E>(fv[u]);
            st16_cg(stage_r + a.stage_stride + g * WB, U::encode(fv[u]));
          } else if (g + E <= P) {
#pragma unroll
            for (int q = 0; q < E; q += 4)
              st16_f(a.v[lr] + g + q, make_float4(fv[u][q], fv[u][q + 1], fv[u][q + 2], fv[u][q + 3]));
          } else {
#pragma unroll
            for (int q = 0; q < E; ++q)
              if (g + q < P) a.v[lr][g + q] = fv[u][q];
          }
        }
        st |= unit_status<W16, E>(f[u]);
        st16_cg(stage_r + g * WB, U::encode(f[u]));
      }
    }
  }
}

// a2 for one wire unit of ONE segment: E elements at global offset g (a unit
// never straddles two segments: L is a multiple of 256).  Same arithmetic as
// precast_unit; the one-shot kernel spreads (segment, unit) pairs over its
// threads, so a small chunk keeps every thread busy with independent loads.
template <bool W16, bool SGD>
__device__ __forceinline__ void precast_seg_unit(const ExchangeArgs& a, int lr, int64_t g, char* stage_r,
                                                 uint32_t& st) {
  using U = Unit<W16>;
  constexpr int E = U::kElems;
  constexpr int WB = W16 ? 2 : 4;
  const float* __restrict__ x = a.x[lr];
  const int64_t P = a.P;
  float f[E], fv[SGD ? E : 1], fg[SGD ? E : 1];
  if (g + E <= P) {
#pragma unroll
    for (int q = 0; q < E; q += 4) {
      const float4 t = ld16_f(x + g + q);
      f[q] = t.x; f[q + 1] = t.y; f[q + 2] = t.z; f[q + 3] = t.w;
      if constexpr (SGD) {
        const float4 tv = ld16_f(a.v[lr] + g + q), tg = ld16_f(a.g[lr] + g + q);
        fv[q] = tv.x; fv[q + 1] = tv.y; fv[q + 2] = tv.z; fv[q + 3] = tv.w;
        fg[q] = tg.x; fg[q + 1] = tg.y; fg[q + 2] = tg.z; fg[q + 3] = tg.w;
      }
    }
  } else {
#pragma unroll
    for (int q = 0; q < E; ++q) {
      const bool in = g + q < P;
      f[q] = in ? x[g + q] : 0.0f;
      if constexpr (SGD) {
        fv[q] = in ? a.v[lr][g + q] : 0.0f;
        fg[q] = in ? a.g[lr][g + q] : 0.0f;
      }
    }
  }
  if constexpr (SGD) {
#pragma unroll
    for (int q = 0; q < E; ++q) {
      fv[q] = g + q < P ? sgd_v1(fv[q], fg[q], a.lr, a.mu) : 0.0f;
      f[q] = g + q < P ? __fadd_rn(f[q], fv[q]) : 0.0f;
    }
    if (a.nvec == 2) {  // momentum exchanged: v' goes to the wire (vector 1)
      st |= unit_status<W16, E>(fv);
      st16_cg(stage_r + a.stage_stride + g * WB, U::encode(fv));
    } else if (g + E <= P) {
#pragma unroll
      for (int q = 0; q < E; q += 4) st16_f(a.v[lr] + g + q, make_float4(fv[q], fv[q + 1], fv[q + 2], fv[q + 3]));
    } else {
#pragma unroll
      for (int q = 0; q < E; ++q)
        if (g + q < P) a.v[lr][g + q] = fv[q];
    }
  }
  st |= unit_status<W16, E>(f);
  st16_cg(stage_r + g * WB, U::encode(f));
}

template <int K, bool W16, bool SYS, bool SGD>
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
    uint32_t* ctr = a.flags[r] + (size_t)kPhases * TM_MAX_RANKS * a.flag_stride + c;
    s_epoch = *ctr + 1;
    *ctr = s_epoch;
  }
  __syncthreads();
  const uint32_t epoch = s_epoch;
  stamp(a, kStampStart);
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
  for (int v = threadIdx.x; v < nu32; v += kThreads) {
    const int64_t ev = e0 + (int64_t)v * E;
    precast_unit<W16, K, SGD>(a, lr, ev, stage_r, st);
  }
  if (st) atomicOr(a.status, st);  // rare: only threads that saw a bad value
  stamp(a, kStampCast);

  if (!rank_barrier<K, SYS>(a, kPhaseReady, r, c, epoch, &s_abort)) return;
  stamp(a, kStampReady);

  // ---------------- a4: reduce-scatter pull, fused sum / (1/k) / cast -------
  for (int vq = 0; vq < a.nvec; ++vq) {
    const char* src[K];
#pragma unroll
    for (int j = 0; j < K; ++j) src[j] = reinterpret_cast<const char*>(a.stage[j]) + vq * a.stage_stride;
    char* const avg_r = reinterpret_cast<char*>(a.avg[r]) + vq * a.avg_stride;
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
      if (!a.sum) {
#pragma unroll
        for (int q = 0; q < E; ++q) s[q] = div_k<K>(s[q]);
      } else if (W16) {  // a sum can leave the binary16 range
#pragma unroll
        for (int q = 0; q < E; ++q) st |= status_of(s[q], true) & TM_BIT_OVERFLOW16;
      }
      st16_cg(avg_r + (e0 + v * E) * WB, U::encode(s));
    }
  }
  if (st) atomicOr(a.status, st);
  stamp(a, kStampReduce);

  if (!rank_barrier<K, SYS>(a, kPhaseReduced, r, c, epoch, &s_abort)) return;
  stamp(a, kStampReduced);
  if (a.ag_external) return;  // a6 by the copy engines / NCCL (tm_allgather)

  // ---------------- a6: allgather pull, fused widen, store to caller ---------
  for (int vq = 0; vq < a.nvec; ++vq) {
    constexpr int G = K;  // all k owners' units in flight at once
    float* __restrict__ x = vq ? a.v[lr] : a.x[lr];
    for (int v = threadIdx.x; v < nu32; v += kThreads) {
      const int64_t ev = e0 + (int64_t)v * E;
      uint4 raw[G];
#pragma unroll
      for (int j = 0; j < G; ++j)
        raw[j] = ld16_cg(reinterpret_cast<const char*>(a.avg[j]) + vq * a.avg_stride + ev * WB);
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
  stamp(a, kStampEnd);
}

// ---------------------------------------------------------------------------
// Warp-specialised staged kernel: the pre-cast (HBM-bound) overlaps the
// reduce-scatter pull (NVLink-bound across GPUs).  512 threads per CTA: warps
// 0-7 are casters, warps 8-15 reducers.  The CTA's chunk is split into kWsSub
// sub-chunks; the casters pre-cast sub-chunk t of all k segments, sync among
// themselves (named barrier 1) and publish READY_t to every rank, then move on
// to t+1; the reducers wait for READY_t from every rank (named barrier 2) and
// pull / sum / store sub-chunk t of the own segment while the casters work on
// t+1.  After the last sub-chunk the whole CTA meets, publishes REDUCED and runs
// the allgather pull with all 16 warps.  Reuse across exchanges is covered by the
// same argument as the other kernels (READY_t(n+1) is published after AG(n);
// stage is rewritten only after REDUCED(n) from every rank).
// ---------------------------------------------------------------------------
constexpr int kWsThreads = 512;
constexpr int kWsGroup = 256;

__device__ __forceinline__ void named_bar(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

template <int K, bool W16, bool SYS, bool SGD>
__global__ void __launch_bounds__(kWsThreads, 2)
tm_exchange_ws_kernel(const __grid_constant__ ExchangeArgs a) {
  using U = Unit<W16>;
  constexpr int E = U::kElems;
  constexpr int WB = W16 ? 2 : 4;
  __shared__ int s_abort;
  __shared__ uint32_t s_epoch;

  const int lr = blockIdx.x / a.C;
  const int c = blockIdx.x - lr * a.C;
  const int r = a.rank0 + lr;
  if (threadIdx.x == 0) {
    s_abort = 0;
    uint32_t* ctr = a.flags[r] + (size_t)kPhases * TM_MAX_RANKS * a.flag_stride + c;
    s_epoch = *ctr + 1;
    *ctr = s_epoch;
  }
  __syncthreads();
  const uint32_t epoch = s_epoch;
  stamp(a, kStampStart);
  const int64_t P = a.P, L = a.L;
  const int64_t e0 = (int64_t)c * a.Lc;
  const int64_t e1 = min(e0 + a.Lc, L);
  const int64_t nel = e1 > e0 ? e1 - e0 : 0;
  const int nsub = (int)max((int64_t)1, min((int64_t)kWsSub, nel / kWsMinSub));  // same on every rank
  const int64_t Ls = ((nel + nsub - 1) / nsub + 255) / 256 * 256;  // sub-chunk length
  char* const stage_r = reinterpret_cast<char*>(a.stage[r]);
  const int grp = threadIdx.x / kWsGroup;
  const int tg = threadIdx.x - grp * kWsGroup;
  uint32_t st = 0;

  if (grp == 0) {
    // ------------------------------------------------ casters: a2 per sub-chunk
    for (int t = 0; t < nsub; ++t) {
      const int64_t s0e = e0 + (int64_t)t * Ls;
      const int64_t s1e = min(s0e + Ls, e1);
      const int nu = s1e > s0e ? (int)((s1e - s0e) / E) : 0;
      for (int v = tg; v < nu; v += kWsGroup) {
        const int64_t ev = s0e + (int64_t)v * E;
        precast_unit<W16, K, SGD>(a, lr, ev, stage_r, st);
      }
      named_bar(1, kWsGroup);  // every caster's stage writes of sub-chunk t done
      if (tg < K)
        st_release<SYS>(a.flags[tg] + (size_t)(t * TM_MAX_RANKS + r) * a.flag_stride + c, epoch);
    }
  } else {
    // ------------------------------------------------ reducers: a4 per sub-chunk
    for (int t = 0; t < nsub; ++t) {
      if (tg < K) {  // READY_t from rank tg
        const uint32_t* mine = a.flags[r] + (size_t)(t * TM_MAX_RANKS + tg) * a.flag_stride + c;
        if ((int32_t)(ld_acquire<SYS>(mine) - epoch) < 0) {
          const uint64_t t0 = globaltimer();
          while ((int32_t)(ld_acquire<SYS>(mine) - epoch) < 0) {
            if (globaltimer() - t0 > a.timeout_ns) {
              atomicOr(a.status, TM_BIT_TIMEOUT);
              s_abort = 1;
              break;
            }
            __nanosleep(32);
          }
        }
      }
      named_bar(2, kWsGroup);
      if (s_abort) break;
      const int64_t s0e = e0 + (int64_t)t * Ls;
      const int64_t s1e = min(s0e + Ls, e1);
      const int nu = s1e > s0e ? (int)((s1e - s0e) / E) : 0;
      for (int vw = tg; vw < nu * a.nvec; vw += kWsGroup) {
        const int vq = vw >= nu;  // vector of this unit (0: w / x, 1: v)
        const int v = vw - vq * nu;
        const char* src[K];
#pragma unroll
        for (int j = 0; j < K; ++j) src[j] = reinterpret_cast<const char*>(a.stage[j]) + vq * a.stage_stride;
        char* const avg_r = reinterpret_cast<char*>(a.avg[r]) + vq * a.avg_stride;
        const int64_t e = s0e + (int64_t)v * E;
        const int64_t off = ((int64_t)r * L + e) * WB;
        uint4 raw[K];
#pragma unroll
        for (int j = 0; j < K; ++j) raw[j] = ld16_cg(src[j] + off);
        float sm[E], tt[E];
        U::decode(raw[0], sm);
#pragma unroll
        for (int j = 1; j < K; ++j) {
          U::decode(raw[j], tt);
#pragma unroll
          for (int q = 0; q < E; ++q) sm[q] = __fadd_rn(sm[q], tt[q]);
        }
        if (!a.sum) {
#pragma unroll
          for (int q = 0; q < E; ++q) sm[q] = div_k<K>(sm[q]);
        } else if (W16) {
#pragma unroll
          for (int q = 0; q < E; ++q) st |= status_of(sm[q], true) & TM_BIT_OVERFLOW16;
        }
        st16_cg(avg_r + e * WB, U::encode(sm));
      }
    }
  }
  if (st) atomicOr(a.status, st);
  __syncthreads();
  if (s_abort) return;
  stamp(a, kStampReduce);  // pre-cast and reduce-scatter overlap: one stamp for both
  if (!rank_barrier<K, SYS>(a, kWsSub, r, c, epoch, &s_abort)) return;  // REDUCED
  stamp(a, kStampReduced);
  if (a.ag_external) return;  // a6 by the copy engines / NCCL (tm_allgather)

  // ---------------- a6: allgather pull with all 16 warps ----------------------
  const int nu32 = (int)(nel / E);
  for (int vw = threadIdx.x; vw < nu32 * a.nvec; vw += kWsThreads) {
    const int vq = vw >= nu32;
    const int v = vw - vq * nu32;
    float* __restrict__ x = vq ? a.v[lr] : a.x[lr];
    const int64_t ev = e0 + (int64_t)v * E;
    uint4 raw[K];
#pragma unroll
    for (int j = 0; j < K; ++j)
      raw[j] = ld16_cg(reinterpret_cast<const char*>(a.avg[j]) + vq * a.avg_stride + ev * WB);
#pragma unroll
    for (int j = 0; j < K; ++j) {
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
  stamp(a, kStampEnd);
}

// ---------------------------------------------------------------------------
// The same three phases on the TMA engine (default staged kernel).
//
// One CTA per SM (224 KB of shared memory).  Each phase is a tile pipeline:
// thread 0 issues 1-D bulk copies (cp.async.bulk, completing on an mbarrier)
// of the phase's source tiles into a 4-slot x 32 KB input ring -- for a4 the k
// sources are peer staging buffers, i.e. the TMA engine pulls over NVLink --
// all threads transform the tile in shared memory into a 3-slot x 32 KB output
// ring, and thread 0 bulk-stores it.  Bytes in flight are set by the rings, not
// by registers or LSU queue depth (the register kernel above was lg_throttle-
// bound).  Cross-proxy ordering: before a phase's flags are released, thread 0
// waits for its bulk stores to complete and issues fence.proxy.async.global;
// after a barrier it fences again before issuing bulk loads of peer data.
// Elements in [P & ~3, P) (at most 3, in the last segment) are read / written
// with plain accesses; elements >= P are zero on the wire and never stored.
// ---------------------------------------------------------------------------
constexpr int kSlotBytes = 32 * 1024;
constexpr int kInSlots = 4;
constexpr int kOutSlots = 3;
constexpr int kTmaThreads = 512;  // 16 warps share the in-smem transform of each tile

__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

// A group of NT threads that runs tile pipelines together: the whole CTA
// (BAR = 0, __syncthreads) or half of it (named barrier BAR), with NIN input
// slots of INB bytes and NOUT output slots of OUTB bytes.
template <int NT, int BAR, int NIN, int NOUT, int INB, int OUTB>
struct Grp {
  static constexpr int kNT = NT, kNin = NIN, kNout = NOUT, kInB = INB, kOutB = OUTB;
  __device__ static void sync() {
    if constexpr (BAR == 0) __syncthreads();
    else named_bar(BAR, NT);
  }
};
using FullGrp = Grp<kTmaThreads, 0, kInSlots, kOutSlots, kSlotBytes, kSlotBytes>;

// Runs n_items through the group's rings.  issue(i, slot, bar) [group thread 0]
// starts the bulk loads of item i and arms `bar` with their byte count;
// compute(i, in, out) [all group threads] transforms; store(i, out) [group
// thread 0] issues the bulk stores.  `use` / `outn` continue across calls so
// slot parities stay consistent.
// Wait for a ring slot whose bulk copies may read PEER memory (NVLink): a copy
// that never completes must not hang the box, so after the barrier timeout the
// wait sets TM_BIT_TIMEOUT and traps (the launch fails with an error the host
// sees, instead of spinning forever).
__device__ __forceinline__ void mbar_wait_bounded(uint64_t* bar, uint32_t parity, uint64_t timeout_ns,
                                                  uint32_t* status) {
  const uint32_t a = smem_u32(bar);
  uint32_t done = 0;
  asm volatile(
      "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(done) : "r"(a), "r"(parity) : "memory");
  if (done) return;
  const uint64_t t0 = globaltimer();
  for (;;) {
    asm volatile(
        "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done) : "r"(a), "r"(parity) : "memory");
    if (done) return;
    if (globaltimer() - t0 > timeout_ns) {
      atomicOr(status, TM_BIT_TIMEOUT);
      __threadfence_system();
      __trap();
    }
  }
}

template <class G, class IssueF, class ComputeF, class StoreF>
__device__ __forceinline__ void tile_pipeline(int gtid, int n_items, uint32_t& use, uint32_t& outn,
                                              char* in_ring, char* out_ring, uint64_t* full,
                                              IssueF issue, ComputeF compute, StoreF store,
                                              uint64_t timeout_ns, uint32_t* status) {
  if (gtid == 0) {
    for (int i = 0; i < G::kNin && i < n_items; ++i) {
      const uint32_t slot = (use + i) % G::kNin;
      issue(i, in_ring + slot * G::kInB, &full[slot]);
    }
  }
  for (int i = 0; i < n_items; ++i) {
    const uint32_t u = use + i;
    const uint32_t slot = u % G::kNin;
    mbar_wait_bounded(&full[slot], (u / G::kNin) & 1, timeout_ns, status);
    char* out = out_ring + (outn % G::kNout) * G::kOutB;
    compute(i, in_ring + slot * G::kInB, out);
    fence_proxy_async_smem();                             // generic smem writes -> bulk store
    if (gtid == 0) bulk_wait_read<G::kNout - 2>();        // out slot of item i+1 is free
    G::sync();                                            // every thread is done with slot / out
    if (gtid == 0) {
      store(i, out);
      bulk_commit();
      if (i + G::kNin < n_items) issue(i + G::kNin, in_ring + slot * G::kInB, &full[slot]);
    }
    ++outn;
  }
  use += n_items;
}

// Wait for this thread's bulk stores and order them before a generic-proxy release.
__device__ __forceinline__ void drain_bulk_stores_thread() {
  bulk_wait_all<0>();
  fence_proxy_async_global();
}

// What the phases of one CTA need to know.
struct PhaseCtx {
  const ExchangeArgs* a;
  int lr, r;
  float* x;
  int64_t P, L, P4;
  char* stage_r;
};

// a2 on the TMA engine: pre-cast the chunk range [s0, s1) of all K segments into
// the own stage.  Fused BSP step (SGD): the tile is TPS elements of w, v and g
// (three bulk loads into one slot); v' goes back to v with register stores
// (1.819 vs 1.835 ms for a second bulk store from the output slot), the wire
// tile of w' = w + v' is bulk-stored as in the plain pre-cast.
template <class G, int K, bool W16, bool SGD>
__device__ __forceinline__ void precast_phase(const PhaseCtx& pc, int gtid, int64_t s0, int64_t s1,
                                              uint32_t& use, uint32_t& outn, char* in_ring,
                                              char* out_ring, uint64_t* full, uint32_t& st) {
  using U = Unit<W16>;
  constexpr int E = U::kElems;
  constexpr int WB = W16 ? 2 : 4;
  constexpr int TP = G::kInB / 4;                 // plain tile: fp32 in one input slot
  constexpr int TPS = G::kInB / 16;               // SGD tile: w, v, g in one input slot (2048 for 32 KB: 1.82 ms vs 1.87 for 2560)
  static_assert(TP * WB <= G::kOutB && TPS >= 256 && 2 * TPS * WB <= G::kOutB, "pre-cast tiles");
  const ExchangeArgs& a = *pc.a;
  const int tp = SGD ? TPS : TP;
  float* const x = pc.x;
  float* const vr = a.v[pc.lr];
  const float* const gr = a.g[pc.lr];
  const int64_t P = pc.P, L = pc.L, P4 = pc.P4;
  const int64_t nel = s1 > s0 ? s1 - s0 : 0;
  const int nt = (int)((nel + tp - 1) / tp);
  auto geom = [&](int i, int64_t& g0, int64_t& n) {
    const int sg = i / nt, t = i - sg * nt;
    g0 = (int64_t)sg * L + s0 + (int64_t)t * tp;
    n = min((int64_t)tp, nel - (int64_t)t * tp);
  };
  tile_pipeline<G>(
      gtid, K * nt, use, outn, in_ring, out_ring, full,
      [&](int i, char* slot, uint64_t* bar) {
        int64_t g0, n;
        geom(i, g0, n);
        const int64_t nb = max((int64_t)0, min(g0 + n, P4) - g0);  // bulk-loadable elements
        mbar_expect_tx(bar, (uint32_t)(nb * 4 * (SGD ? 3 : 1)));
        if (nb > 0) {
          bulk_load(slot, x + g0, (uint32_t)(nb * 4), bar);
          if (SGD) {
            bulk_load(slot + TPS * 4, vr + g0, (uint32_t)(nb * 4), bar);
            bulk_load(slot + 2 * TPS * 4, gr + g0, (uint32_t)(nb * 4), bar);
          }
        }
      },
      [&](int i, const char* in, char* out) {
        int64_t g0, n;
        geom(i, g0, n);
        const int nbi = (int)max((int64_t)0, min(g0 + n, P4) - g0);
        const float* fin = reinterpret_cast<const float*>(in);
        const float* fvin = fin + TPS;
        const float* fgin = fin + 2 * TPS;
        const bool mom = SGD && a.nvec == 2;  // v' to the wire (second output tile), not back to v
        uint4* out2 = reinterpret_cast<uint4*>(out + TPS * WB);
        for (int v = gtid; v < (int)(n / E); v += G::kNT) {
          float f[E], f2[SGD ? E : 1];
          if ((v + 1) * E <= nbi) {
#pragma unroll
            for (int q = 0; q < E; q += 4) {
              float4 t4 = reinterpret_cast<const float4*>(fin + v * E)[q / 4];
              if (SGD) {
                const float4 vn = sgd_v(reinterpret_cast<const float4*>(fvin + v * E)[q / 4],
                                        reinterpret_cast<const float4*>(fgin + v * E)[q / 4], a.lr, a.mu);
                if (mom) {
                  f2[q] = vn.x; f2[q + 1] = vn.y; f2[q + 2] = vn.z; f2[q + 3] = vn.w;
                } else {
                  st16_f(vr + g0 + v * E + q, vn);
                }
                t4 = add4(t4, vn);
              }
              f[q] = t4.x; f[q + 1] = t4.y; f[q + 2] = t4.z; f[q + 3] = t4.w;
            }
          } else {
#pragma unroll
            for (int q = 0; q < E; ++q) {
              const int e = v * E + q;
              if (SGD) f2[q] = 0.0f;
              if (e < nbi) {
                f[q] = fin[e];
                if (SGD) {
                  const float vn = sgd_v1(fvin[e], fgin[e], a.lr, a.mu);
                  if (mom) f2[q] = vn;
                  else vr[g0 + e] = vn;
                  f[q] = __fadd_rn(f[q], vn);
                }
              } else if (g0 + e < P) {  // the <= 3 elements in [P & ~3, P): plain accesses
                f[q] = x[g0 + e];
                if (SGD) {
                  const float vn = sgd_v1(vr[g0 + e], gr[g0 + e], a.lr, a.mu);
                  if (mom) f2[q] = vn;
                  else vr[g0 + e] = vn;
                  f[q] = __fadd_rn(f[q], vn);
                }
              } else {
                f[q] = 0.0f;
              }
            }
          }
          st |= unit_status<W16, E>(f);
          reinterpret_cast<uint4*>(out)[v] = U::encode(f);
          if constexpr (SGD) {
            if (mom) {
              st |= unit_status<W16, E>(f2);
              out2[v] = U::encode(f2);
            }
          }
        }
      },
      [&](int i, const char* out) {
        int64_t g0, n;
        geom(i, g0, n);
        bulk_store(pc.stage_r + g0 * WB, out, (uint32_t)(n * WB));
        if (SGD && a.nvec == 2)
          bulk_store(pc.stage_r + a.stage_stride + g0 * WB, out + TPS * WB, (uint32_t)(n * WB));
      },
      a.timeout_ns, a.status);
}

// a4 on the TMA engine: pull [s0, s1) of the own segment from every rank's
// stage (peer memory), ascending-rank fp32 sum, 1/k, round, store into own avg.
template <class G, int K, bool W16>
__device__ __forceinline__ void reduce_phase(const PhaseCtx& pc, int gtid, int64_t s0, int64_t s1,
                                             uint32_t& use, uint32_t& outn, char* in_ring,
                                             char* out_ring, uint64_t* full, uint32_t& st, int vq = 0) {
  using U = Unit<W16>;
  constexpr int E = U::kElems;
  constexpr int WB = W16 ? 2 : 4;
  // k sources of TR wire elements fit one input slot; a multiple of 256 elements
  // keeps every source's smem offset and byte count 16-byte aligned.
  constexpr int TR_RAW = G::kInB / (K * WB) / 256 * 256;
  constexpr int TR = TR_RAW < 4096 ? TR_RAW : 4096;
  static_assert(TR >= 256 && TR * WB <= G::kOutB, "a4 tile");
  const ExchangeArgs& a = *pc.a;
  const int r = pc.r;
  const int64_t L = pc.L;
  char* const avg_r = reinterpret_cast<char*>(a.avg[r]) + vq * a.avg_stride;
  const int64_t soff = vq * a.stage_stride;  // vector vq's staging
  const int nt = (int)((max((int64_t)0, s1 - s0) + TR - 1) / TR);
  tile_pipeline<G>(
      gtid, nt, use, outn, in_ring, out_ring, full,
      [&](int i, char* slot, uint64_t* bar) {
        const int64_t e = s0 + (int64_t)i * TR;
        const int64_t n = min((int64_t)TR, s1 - e);
        mbar_expect_tx(bar, (uint32_t)(K * n * WB));
#pragma unroll
        for (int j = 0; j < K; ++j)
          bulk_load(slot + j * TR * WB,
                    reinterpret_cast<const char*>(a.stage[j]) + soff + ((int64_t)r * L + e) * WB,
                    (uint32_t)(n * WB), bar);
      },
      [&](int i, const char* in, char* out) {
        const int64_t e = s0 + (int64_t)i * TR;
        const int n = (int)min((int64_t)TR, s1 - e);
        for (int v = gtid; v < n / E; v += G::kNT) {
          uint4 raw[K];
#pragma unroll
          for (int j = 0; j < K; ++j) raw[j] = reinterpret_cast<const uint4*>(in + j * TR * WB)[v];
          float sm[E], t[E];
          U::decode(raw[0], sm);
#pragma unroll
          for (int j = 1; j < K; ++j) {
            U::decode(raw[j], t);
#pragma unroll
            for (int q = 0; q < E; ++q) sm[q] = __fadd_rn(sm[q], t[q]);
          }
          if (!a.sum) {
#pragma unroll
            for (int q = 0; q < E; ++q) sm[q] = div_k<K>(sm[q]);
          } else if (W16) {  // a sum can leave the binary16 range
#pragma unroll
            for (int q = 0; q < E; ++q) st |= status_of(sm[q], true) & TM_BIT_OVERFLOW16;
          }
          reinterpret_cast<uint4*>(out)[v] = U::encode(sm);
        }
      },
      [&](int i, const char* out) {
        const int64_t e = s0 + (int64_t)i * TR;
        const int64_t n = min((int64_t)TR, s1 - e);
        bulk_store(avg_r + e * WB, out, (uint32_t)(n * WB));
      },
      a.timeout_ns, a.status);
}

// a6 on the TMA engine: pull chunk [e0, e1) of every rank's avg, widen, store
// into the caller's buffer (truncated at P).
template <class G, int K, bool W16>
__device__ __forceinline__ void gather_phase(const PhaseCtx& pc, int gtid, int64_t e0, int64_t e1,
                                             uint32_t& use, uint32_t& outn, char* in_ring,
                                             char* out_ring, uint64_t* full, int vq = 0) {
  using U = Unit<W16>;
  constexpr int E = U::kElems;
  constexpr int WB = W16 ? 2 : 4;
  constexpr int TA = G::kOutB / 4;  // fp32 out tile fills one output slot
  static_assert(TA * WB <= G::kInB, "a6 tile");
  const ExchangeArgs& a = *pc.a;
  float* const x = vq ? a.v[pc.lr] : pc.x;  // vector vq's caller buffer
  const int64_t aoff = vq * a.avg_stride;
  const int64_t P = pc.P, L = pc.L, P4 = pc.P4;
  const int64_t nel = e1 > e0 ? e1 - e0 : 0;
  const int nt = (int)((nel + TA - 1) / TA);
  auto geom = [&](int i, int& j, int64_t& e, int64_t& n) {
    j = i / nt;
    const int t = i - j * nt;
    e = e0 + (int64_t)t * TA;
    n = min((int64_t)TA, e1 - e);
  };
  tile_pipeline<G>(
      gtid, K * nt, use, outn, in_ring, out_ring, full,
      [&](int i, char* slot, uint64_t* bar) {
        int j;
        int64_t e, n;
        geom(i, j, e, n);
        mbar_expect_tx(bar, (uint32_t)(n * WB));
        bulk_load(slot, reinterpret_cast<const char*>(a.avg[j]) + aoff + e * WB, (uint32_t)(n * WB), bar);
      },
      [&](int i, const char* in, char* out) {
        int j;
        int64_t e, n;
        geom(i, j, e, n);
        const int64_t g0 = (int64_t)j * L + e;
        // tile-relative window [lo, hi) of the <= 3 elements in [P & ~3, P):
        // bulk stores cannot cover them, plain stores do
        const int lo = (int)max((int64_t)0, min(n, P4 - g0));
        const int hi = (int)max((int64_t)0, min(n, P - g0));
        float* fo = reinterpret_cast<float*>(out);
        for (int v = gtid; v < (int)(n / E); v += G::kNT) {
          float f[E];
          U::decode(reinterpret_cast<const uint4*>(in)[v], f);
#pragma unroll
          for (int q = 0; q < E; q += 4)
            reinterpret_cast<float4*>(fo + v * E)[q / 4] = make_float4(f[q], f[q + 1], f[q + 2], f[q + 3]);
          if (hi > lo && (v + 1) * E > lo && v * E < hi) {
#pragma unroll
            for (int q = 0; q < E; ++q)
              if (v * E + q >= lo && v * E + q < hi) x[g0 + v * E + q] = f[q];
          }
        }
      },
      [&](int i, const char* out) {
        int j;
        int64_t e, n;
        geom(i, j, e, n);
        const int64_t g0 = (int64_t)j * L + e;
        const int64_t nb = max((int64_t)0, min(g0 + n, P4) - g0);
        if (nb > 0) bulk_store(x + g0, out, (uint32_t)(nb * 4));
      },
      a.timeout_ns, a.status);
}

template <int K, bool W16, bool SYS, bool SGD>
__global__ void __launch_bounds__(kTmaThreads, 1)
tm_exchange_tma_kernel(const __grid_constant__ ExchangeArgs a) {
  extern __shared__ __align__(128) unsigned char smem[];
  char* in_ring = reinterpret_cast<char*>(smem);
  char* out_ring = in_ring + kInSlots * kSlotBytes;
  __shared__ __align__(8) uint64_t full[kInSlots];
  __shared__ int s_abort;
  __shared__ uint32_t s_epoch;

  const int lr = blockIdx.x / a.C;
  const int c = blockIdx.x - lr * a.C;
  const int r = a.rank0 + lr;
  const PhaseCtx pc{&a, lr, r, a.x[lr], a.P, a.L, a.P & ~int64_t(3), reinterpret_cast<char*>(a.stage[r])};
  const int64_t e0 = (int64_t)c * a.Lc;
  const int64_t e1 = min(e0 + a.Lc, a.L);
  const int tid = threadIdx.x;

  if (tid == 0) {
    s_abort = 0;
    uint32_t* ctr = a.flags[r] + (size_t)kPhases * TM_MAX_RANKS * a.flag_stride + c;  // device epoch
    s_epoch = *ctr + 1;
    *ctr = s_epoch;
    for (int i = 0; i < kInSlots; ++i) mbar_init(&full[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const uint32_t epoch = s_epoch;
  stamp(a, kStampStart);
  uint32_t use = 0, outn = 0, st = 0;

  precast_phase<FullGrp, K, W16, SGD>(pc, tid, e0, e1, use, outn, in_ring, out_ring, full, st);
  if (st) atomicOr(a.status, st);
  st = 0;
  if (tid == 0) drain_bulk_stores_thread();
  stamp(a, kStampCast);
  if (!rank_barrier<K, SYS>(a, kPhaseReady, r, c, epoch, &s_abort)) return;
  stamp(a, kStampReady);
  if (tid == 0) fence_proxy_async_global();  // peers' staging, acquired above -> bulk loads

  for (int vq = 0; vq < a.nvec; ++vq)
    reduce_phase<FullGrp, K, W16>(pc, tid, e0, e1, use, outn, in_ring, out_ring, full, st, vq);
  if (st) atomicOr(a.status, st);
  if (tid == 0) drain_bulk_stores_thread();
  stamp(a, kStampReduce);
  if (!rank_barrier<K, SYS>(a, kPhaseReduced, r, c, epoch, &s_abort)) return;
  stamp(a, kStampReduced);
  if (a.ag_external) return;  // a6 by the copy engines / NCCL (tm_allgather)
  if (tid == 0) fence_proxy_async_global();

  for (int vq = 0; vq < a.nvec; ++vq)
    gather_phase<FullGrp, K, W16>(pc, tid, e0, e1, use, outn, in_ring, out_ring, full, vq);
  if (tid == 0) bulk_wait_all<0>();  // kernel exit also waits; explicit for clarity
  stamp(a, kStampEnd);
}

// ---------------------------------------------------------------------------
// Warp-specialised staged kernel on the TMA engine: warps 0-7 (casters) run the
// pre-cast pipeline sub-chunk by sub-chunk and publish READY_t to every rank;
// warps 8-15 (reducers) pull sub-chunk t of the own segment from every rank's
// staging as soon as READY_t is in from all of them.  The HBM-bound pre-cast and
// the NVLink-bound reduce-scatter overlap, both fed by bulk copies (the register
// warp-specialised kernel above does the same with 16-byte loads).  Then the
// whole CTA meets at REDUCED and runs the allgather pipeline.  Same flag phases
// as that kernel (READY_0..3, REDUCED = kWsSub).
// Shared memory (224 KB): phase 1 casters [0, 128 KB) = 2 input + 2 output slots
// of 32 KB, reducers [128, 224 KB) = 2 input slots of 32 KB + 2 output slots of
// 16 KB; the allgather reuses all of it as the full-CTA rings.
// ---------------------------------------------------------------------------
using CastGrp = Grp<kTmaThreads / 2, 1, 2, 2, kSlotBytes, kSlotBytes>;
using RedGrp = Grp<kTmaThreads / 2, 2, 2, 2, kSlotBytes, kSlotBytes / 2>;

template <int K, bool W16, bool SYS, bool SGD>
__global__ void __launch_bounds__(kTmaThreads, 1)
tm_exchange_tmaws_kernel(const __grid_constant__ ExchangeArgs a) {
  extern __shared__ __align__(128) unsigned char smem[];
  char* const base = reinterpret_cast<char*>(smem);
  __shared__ __align__(8) uint64_t full_c[CastGrp::kNin];
  __shared__ __align__(8) uint64_t full_r[RedGrp::kNin];
  __shared__ __align__(8) uint64_t full[kInSlots];
  __shared__ int s_abort;
  __shared__ uint32_t s_epoch;

  const int lr = blockIdx.x / a.C;
  const int c = blockIdx.x - lr * a.C;
  const int r = a.rank0 + lr;
  const PhaseCtx pc{&a, lr, r, a.x[lr], a.P, a.L, a.P & ~int64_t(3), reinterpret_cast<char*>(a.stage[r])};
  const int64_t e0 = (int64_t)c * a.Lc;
  const int64_t e1 = min(e0 + a.Lc, a.L);
  const int64_t nel = e1 > e0 ? e1 - e0 : 0;
  const int nsub = (int)max((int64_t)1, min((int64_t)kWsSub, nel / kWsMinSub));  // same on every rank
  const int64_t Ls = ((nel + nsub - 1) / nsub + 255) / 256 * 256;  // sub-chunk length
  const int tid = threadIdx.x;
  constexpr int NT = CastGrp::kNT;
  const int grp = tid / NT;
  const int gtid = tid - grp * NT;

  if (tid == 0) {
    s_abort = 0;
    uint32_t* ctr = a.flags[r] + (size_t)kPhases * TM_MAX_RANKS * a.flag_stride + c;  // device epoch
    s_epoch = *ctr + 1;
    *ctr = s_epoch;
    for (int i = 0; i < CastGrp::kNin; ++i) mbar_init(&full_c[i], 1);
    for (int i = 0; i < RedGrp::kNin; ++i) mbar_init(&full_r[i], 1);
    for (int i = 0; i < kInSlots; ++i) mbar_init(&full[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const uint32_t epoch = s_epoch;
  stamp(a, kStampStart);
  uint32_t st = 0;

  if (grp == 0) {
    // ------------------------------------------------ casters: a2 per sub-chunk
    uint32_t use = 0, outn = 0;
    char* const in_ring = base;
    char* const out_ring = base + CastGrp::kNin * CastGrp::kInB;
    for (int t = 0; t < nsub; ++t) {
      const int64_t s0 = e0 + (int64_t)t * Ls;
      const int64_t s1 = min(s0 + Ls, e1);
      if (s1 > s0)
        precast_phase<CastGrp, K, W16, SGD>(pc, gtid, s0, s1, use, outn, in_ring, out_ring, full_c, st);
      if (gtid == 0) drain_bulk_stores_thread();  // this sub-chunk's staging is in memory
      named_bar(1, NT);
      if (gtid < K)
        st_release<SYS>(a.flags[gtid] + (size_t)(t * TM_MAX_RANKS + r) * a.flag_stride + c, epoch);
    }
  } else {
    // ------------------------------------------------ reducers: a4 per sub-chunk
    uint32_t use = 0, outn = 0;
    char* const in_ring = base + 2 * CastGrp::kNin * CastGrp::kInB;
    char* const out_ring = in_ring + RedGrp::kNin * RedGrp::kInB;
    for (int t = 0; t < nsub; ++t) {
      if (gtid < K) {  // READY_t from rank gtid
        const uint32_t* mine = a.flags[r] + (size_t)(t * TM_MAX_RANKS + gtid) * a.flag_stride + c;
        if ((int32_t)(ld_acquire<SYS>(mine) - epoch) < 0) {
          const uint64_t t0 = globaltimer();
          while ((int32_t)(ld_acquire<SYS>(mine) - epoch) < 0) {
            if (globaltimer() - t0 > a.timeout_ns) {
              atomicOr(a.status, TM_BIT_TIMEOUT);
              s_abort = 1;
              break;
            }
            __nanosleep(32);
          }
        }
      }
      named_bar(2, NT);
      if (s_abort) break;
      if (gtid == 0) fence_proxy_async_global();  // acquired peers' staging -> bulk loads
      const int64_t s0 = e0 + (int64_t)t * Ls;
      const int64_t s1 = min(s0 + Ls, e1);
      if (s1 > s0)
        for (int vq = 0; vq < a.nvec; ++vq)
          reduce_phase<RedGrp, K, W16>(pc, gtid, s0, s1, use, outn, in_ring, out_ring, full_r, st, vq);
    }
    if (gtid == 0) drain_bulk_stores_thread();  // avg in memory before REDUCED
  }
  if (st) atomicOr(a.status, st);
  __syncthreads();
  if (s_abort) return;
  stamp(a, kStampReduce);  // pre-cast and reduce-scatter overlap: one stamp for both
  if (!rank_barrier<K, SYS>(a, kWsSub, r, c, epoch, &s_abort)) return;  // REDUCED
  stamp(a, kStampReduced);
  if (a.ag_external) return;  // a6 by the copy engines / NCCL (tm_allgather)
  if (tid == 0) fence_proxy_async_global();

  // ---------------- a6: allgather pull with the whole CTA ---------------------
  uint32_t use = 0, outn = 0;
  for (int vq = 0; vq < a.nvec; ++vq)
    gather_phase<FullGrp, K, W16>(pc, tid, e0, e1, use, outn, base, base + kInSlots * kSlotBytes, full, vq);
  if (tid == 0) bulk_wait_all<0>();
  stamp(a, kStampEnd);
}

// ---------------------------------------------------------------------------
// One-shot staged kernel (small segments; latency-bound regime): ONE barrier per
// call.  a2 pre-casts chunk c of all k segments into the own staging buffer of
// this call's parity; after READY from every rank, every rank pulls chunk c of
// ALL k segments from ALL k ranks' staging (register loads of peer memory) and
// reduces them itself in ascending rank order, /k, round -- the same arithmetic
// as the owner's a4, so every rank computes bitwise the same average without the
// reduce-scatter / allgather split and without the REDUCED barrier.
// Reuse: staging is double-buffered by the rank's call parity (a per-rank call
// counter in the pad tail: every CTA reads it at start, the last CTA to retire
// increments it, so all CTAs of a launch agree).  Call n writes buffer n & 1;
// the last readers of that buffer are call n-2's, and every rank finished call
// n-2 before it signalled READY(n-1), which this rank acquired in call n-1.
// ---------------------------------------------------------------------------
template <int K, bool W16, bool SYS, bool SGD>
__global__ void __launch_bounds__(kThreads, K == 6 ? 3 : 4)
tm_exchange_oneshot_kernel(const __grid_constant__ ExchangeArgs a) {
  using U = Unit<W16>;
  constexpr int E = U::kElems;
  constexpr int WB = W16 ? 2 : 4;
  __shared__ int s_abort;
  __shared__ uint32_t s_epoch, s_par;

  const int lr = blockIdx.x / a.C;
  const int c = blockIdx.x - lr * a.C;
  const int r = a.rank0 + lr;
  uint32_t* const tail = a.flags[r] + (size_t)(kPhases * TM_MAX_RANKS + 1) * a.flag_stride;
  if (threadIdx.x == 0) {
    s_abort = 0;
    uint32_t* ctr = a.flags[r] + (size_t)kPhases * TM_MAX_RANKS * a.flag_stride + c;
    s_epoch = *ctr + 1;
    *ctr = s_epoch;
    s_par = __ldcg(tail + kTailCalls) & 1u;  // this call's staging parity
    __threadfence();
    // retire: the last of this rank's C CTAs advances the call counter (every CTA
    // has read it by then); the kernel boundary orders it before the next call
    if (atomicAdd(tail + kTailRetire, 1u) == (uint32_t)a.C - 1) {
      tail[kTailRetire] = 0;
      tail[kTailCalls] = __ldcg(tail + kTailCalls) + 1;
    }
  }
  __syncthreads();
  const uint32_t epoch = s_epoch;
  const int64_t boff = (int64_t)s_par * a.nvec_alloc * a.stage_stride;
  stamp(a, kStampStart);
  const int64_t P = a.P, L = a.L;
  const int64_t e0 = (int64_t)c * a.Lc;
  const int64_t e1 = min(e0 + a.Lc, L);
  const int nu = e1 > e0 ? (int)((e1 - e0) / E) : 0;  // wire units per segment chunk
  char* const stage_r = reinterpret_cast<char*>(a.stage[r]) + boff;

  // ---------------- a2: pre-cast chunk c of all k segments (this parity) -------
  // (segment, unit) pairs spread over the threads, unit fastest (coalesced)
  uint32_t st = 0;
  for (int vw = threadIdx.x; vw < nu * K; vw += kThreads) {
    const int sg = vw / nu;
    precast_seg_unit<W16, SGD>(a, lr, (int64_t)sg * L + e0 + (int64_t)(vw - sg * nu) * E, stage_r, st);
  }
  if (st) atomicOr(a.status, st);
  st = 0;
  stamp(a, kStampCast);
  if (!rank_barrier<K, SYS>(a, kPhaseReady, r, c, epoch, &s_abort)) return;
  stamp(a, kStampReady);

  // ---------------- reduce chunk c of EVERY segment from every rank ------------
  for (int vq = 0; vq < a.nvec; ++vq) {
    const char* src[K];
#pragma unroll
    for (int j = 0; j < K; ++j) src[j] = reinterpret_cast<const char*>(a.stage[j]) + boff + vq * a.stage_stride;
    float* __restrict__ x = vq ? a.v[lr] : a.x[lr];
    for (int vw = threadIdx.x; vw < nu * K; vw += kThreads) {  // unit u of segment sg, u fastest
      const int sg = vw / nu;
      const int64_t g = (int64_t)sg * L + e0 + (int64_t)(vw - sg * nu) * E;
      uint4 raw[K];
#pragma unroll
      for (int j = 0; j < K; ++j) raw[j] = ld16_cg(src[j] + g * WB);
      float sm[E], t[E];
      U::decode(raw[0], sm);
#pragma unroll
      for (int j = 1; j < K; ++j) {
        U::decode(raw[j], t);
#pragma unroll
        for (int q = 0; q < E; ++q) sm[q] = __fadd_rn(sm[q], t[q]);
      }
      if (!a.sum) {
#pragma unroll
        for (int q = 0; q < E; ++q) sm[q] = div_k<K>(sm[q]);
      } else if (W16) {  // a sum can leave the binary16 range
#pragma unroll
        for (int q = 0; q < E; ++q) st |= status_of(sm[q], true) & TM_BIT_OVERFLOW16;
      }
      float f[E];
      U::decode(U::encode(sm), f);  // the wire rounding of the average (ASA16: widen(rn16(a)))
      if (g + E <= P) {
        U::store_dst(x + g, f);
      } else {
#pragma unroll
        for (int q = 0; q < E; ++q)
          if (g + q < P) x[g + q] = f[q];
      }
    }
  }
  if (st) atomicOr(a.status, st);
  stamp(a, kStampEnd);
}

// ---------------------------------------------------------------------------
// Low-latency ("LL") staged kernel (small exchanges; latency-bound regime): NO
// barrier and no flag round trip.  Each wire line is 16 bytes {payload word,
// epoch, payload word, epoch}: the epoch travels in the same single-copy-atomic
// 8-byte halves as the data, so a reader that sees the call's epoch in a half
// has that half's data.  Each thread owns a unit of 4 elements end to end:
//   push  load its 4 fp32 elements (or compute w' = w + v' of the fused BSP
//         step), encode them on the wire (ASA16: rn16, one line; ASA: fp32, two
//         lines) and store the line(s) into EVERY rank's receive buffer, slot of
//         the own rank (remote stores over NVLink; the own rank's locally);
//   pull  poll the own receive buffer until the k ranks' lines of this unit
//         carry the call's epoch, then reduce them in ascending rank order, /k,
//         wire rounding (ASA16: widen(rn16(a)), reading R1) and store the unit.
// Bitwise the owner's a4 arithmetic for every element (as the one-shot kernel).
// The epoch is the rank's device call counter + 1 (the one-shot kernel's tail
// counter: every CTA reads it at start, the last to retire increments it) and
// the receive buffers are double-buffered by its parity: call n writes buffer
// n & 1 of every peer, whose previous use was call n-2, finished on that peer
// before it pushed call n-1's lines, which this rank received before starting
// call n.  Stale lines of call n-2 carry epoch n-1 != n+1 and are never taken.
// Receive buffer of rank j (in its staging region): line
//   ((parity * nvec_alloc + vq) * k + src) * LPS + unit * LPU + h
// with LPS = stage_stride / (16 k) lines per source and LPU = 1 (fp16 wire) or
// 2 (fp32 wire) lines per unit.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void st_ll(void* p, uint32_t d0, uint32_t d1, uint32_t ep) {
  asm volatile("st.volatile.global.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(d0), "r"(ep), "r"(d1), "r"(ep)
               : "memory");
}
__device__ __forceinline__ uint4 ld_ll(const void* p) {
  uint4 v;
  asm volatile("ld.volatile.global.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p)
               : "memory");
  return v;
}

template <int K, bool W16, bool SYS, bool SGD>
__global__ void __launch_bounds__(kThreads)
tm_exchange_ll_kernel(const __grid_constant__ ExchangeArgs a) {
  constexpr int LPU = W16 ? 1 : 2;
  __shared__ uint32_t s_calls;
  const int lr = blockIdx.x / a.C;
  const int c = blockIdx.x - lr * a.C;
  const int r = a.rank0 + lr;
  uint32_t* const tail = a.flags[r] + (size_t)(kPhases * TM_MAX_RANKS + 1) * a.flag_stride;
  if (threadIdx.x == 0) {
    s_calls = __ldcg(tail + kTailCalls);
    __threadfence();
    if (atomicAdd(tail + kTailRetire, 1u) == (uint32_t)a.C - 1) {  // as the one-shot kernel
      tail[kTailRetire] = 0;
      tail[kTailCalls] = __ldcg(tail + kTailCalls) + 1;
    }
  }
  __syncthreads();
  const uint32_t epoch = s_calls + 1;
  const int par = (int)(s_calls & 1u);
  stamp(a, kStampStart);
  const int64_t n = a.P;
  const int64_t nu = (n + 3) / 4;
  const int64_t lps = a.stage_stride / (16 * (int64_t)a.k);
  const int64_t stride = (int64_t)a.C * kThreads;
  float* const x = a.x[lr];
  uint32_t st = 0;
  bool late = false;
  for (int64_t u = (int64_t)c * kThreads + threadIdx.x; u < nu; u += stride) {
    const int64_t g = u * 4;
    // ---------------- push: encode the unit, store it into every rank's buffer
    float f[4], fv[4];
    if (g + 4 <= n) {
      const float4 t = ld16_f(x + g);
      f[0] = t.x; f[1] = t.y; f[2] = t.z; f[3] = t.w;
    } else {
#pragma unroll
      for (int q = 0; q < 4; ++q) f[q] = g + q < n ? x[g + q] : 0.0f;
    }
    if constexpr (SGD) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        fv[q] = g + q < n ? sgd_v1(a.v[lr][g + q], a.g[lr][g + q], a.lr, a.mu) : 0.0f;
        f[q] = g + q < n ? __fadd_rn(f[q], fv[q]) : 0.0f;
      }
      if (a.nvec == 1) {  // v' back to v (the momentum is not exchanged)
#pragma unroll
        for (int q = 0; q < 4; ++q)
          if (g + q < n) a.v[lr][g + q] = fv[q];
      } else {
        st |= unit_status<W16, 4>(fv);
      }
    }
    st |= unit_status<W16, 4>(f);
    for (int vq = 0; vq < a.nvec; ++vq) {
      const float* src = (SGD && vq == 1) ? fv : f;
      uint32_t w[2 * LPU];
      if constexpr (W16) {
        w[0] = pack_rn16x2(src[0], src[1]);
        w[1] = pack_rn16x2(src[2], src[3]);
      } else {
#pragma unroll
        for (int q = 0; q < 4; ++q) w[q] = __float_as_uint(src[q]);
      }
      const int64_t line = ((int64_t)(par * a.nvec_alloc + vq) * a.k + r) * lps + u * LPU;
#pragma unroll
      for (int j = 0; j < K; ++j) {
        char* dst = reinterpret_cast<char*>(a.stage[j]) + line * 16;
#pragma unroll
        for (int h = 0; h < LPU; ++h) st_ll(dst + h * 16, w[2 * h], w[2 * h + 1], epoch);
      }
    }
    // ---------------- pull: the k ranks' lines of this unit, rank order
    for (int vq = 0; vq < a.nvec; ++vq) {
      const char* base = reinterpret_cast<const char*>(a.stage[r]) +
                         (((int64_t)(par * a.nvec_alloc + vq) * a.k) * lps + u * LPU) * 16;
      uint4 ln[K][LPU];
      uint32_t ready = 0;  // bit j: rank j's line(s) in
      uint64_t t0 = 0;
      for (int spin = 0; ready != (1u << K) - 1u && !late; ++spin) {
#pragma unroll
        for (int j = 0; j < K; ++j) {
          if (!(ready >> j & 1u)) {
            bool ok = true;
#pragma unroll
            for (int h = 0; h < LPU; ++h) {
              ln[j][h] = ld_ll(base + ((int64_t)j * lps + h) * 16);
              ok = ok && ln[j][h].y == epoch && ln[j][h].w == epoch;
            }
            if (ok) ready |= 1u << j;
          }
        }
        if (ready != (1u << K) - 1u && (spin & 63) == 63) {
          const uint64_t now = globaltimer();
          if (t0 == 0) t0 = now;
          else if (now - t0 > a.timeout_ns) late = true;
        }
      }
      if (late) break;
      float sm[4], t[4];
#pragma unroll
      for (int j = 0; j < K; ++j) {
        if constexpr (W16) {
          const float2 lo = unpack16x2(ln[j][0].x), hi = unpack16x2(ln[j][0].z);
          t[0] = lo.x; t[1] = lo.y; t[2] = hi.x; t[3] = hi.y;
        } else {
          t[0] = __uint_as_float(ln[j][0].x); t[1] = __uint_as_float(ln[j][0].z);
          t[2] = __uint_as_float(ln[j][LPU - 1].x); t[3] = __uint_as_float(ln[j][LPU - 1].z);
        }
        if (j == 0) {
#pragma unroll
          for (int q = 0; q < 4; ++q) sm[q] = t[q];
        } else {
#pragma unroll
          for (int q = 0; q < 4; ++q) sm[q] = __fadd_rn(sm[q], t[q]);
        }
      }
      if (!a.sum) {
#pragma unroll
        for (int q = 0; q < 4; ++q) sm[q] = div_k<K>(sm[q]);
      } else if (W16) {  // a sum can leave the binary16 range
#pragma unroll
        for (int q = 0; q < 4; ++q) st |= status_of(sm[q], true) & TM_BIT_OVERFLOW16;
      }
      if constexpr (W16) {  // the wire rounding of the average: widen(rn16(a))
        const float2 lo = unpack16x2(pack_rn16x2(sm[0], sm[1])), hi = unpack16x2(pack_rn16x2(sm[2], sm[3]));
        sm[0] = lo.x; sm[1] = lo.y; sm[2] = hi.x; sm[3] = hi.y;
      }
      float* dstx = vq ? a.v[lr] : x;
      if (g + 4 <= n) {
        st16_f(dstx + g, make_float4(sm[0], sm[1], sm[2], sm[3]));
      } else {
#pragma unroll
        for (int q = 0; q < 4; ++q)
          if (g + q < n) dstx[g + q] = sm[q];
      }
    }
    if (late) break;
  }
  if (late) st |= TM_BIT_TIMEOUT;
  if (st) atomicOr(a.status, st);
  // push and pull are fused per unit (no phase boundary): the intermediate
  // phase stamps all mark the end of the fused loop
  stamp(a, kStampCast);
  stamp(a, kStampReady);
  stamp(a, kStampReduce);
  stamp(a, kStampReduced);
  stamp(a, kStampEnd);
}

// ---------------------------------------------------------------------------
// Two-shot LL kernel ("LL2", mid-size exchanges): the ASA split of Fig. 2 with
// epoch-tagged lines instead of barriers.  Per call, each thread runs
//   A  push: for every unit (4 elements) of the own buffer it is assigned,
//      encode it (wire rounding) and store its line(s) into the OWNER's
//      reduce-scatter buffer, slot of the own rank (one remote store per unit);
//   B  reduce: for every unit of the own segment it is assigned, poll the k
//      ranks' lines, sum in ascending rank order, /k, round to the wire, and
//      store the averaged line(s) into EVERY rank's allgather buffer, slot of
//      the own segment (the fused a4 + a6 push);
//   C  pull: for every unit of the own buffer it is assigned, poll the owner's
//      averaged line and widen it into the caller's buffer.
// Every thread finishes all its A before any B, and all its B before any C, so
// no thread waits on a line another thread only writes after waiting itself.
// Bitwise the owner's a4 arithmetic (same result as every flavour).  Reuse by
// the device call parity (as LL): rank r writes owner s's reduce-scatter slot
// in call n only after its call n-1 received s's averaged lines of call n-1,
// which s pushed after finishing call n-2; owner s writes rank j's allgather
// slot in call n only after receiving j's call-n lines, i.e. after j finished
// call n-2.  Layout of rank j's receive region per (parity, vector): [RS: k
// source slots][AG: k owner slots] of LPG lines each, LPG = stage_stride /
// (32 k), LPU lines per unit (1 fp16 wire, 2 fp32).
// ---------------------------------------------------------------------------
template <int LPU>
__device__ __forceinline__ bool poll_lines(const char* p, uint32_t epoch, uint4 (&ln)[LPU], uint64_t timeout_ns) {
  uint64_t t0 = 0;
  for (int spin = 0;; ++spin) {
    bool ok = true;
#pragma unroll
    for (int h = 0; h < LPU; ++h) {
      ln[h] = ld_ll(p + h * 16);
      ok = ok && ln[h].y == epoch && ln[h].w == epoch;
    }
    if (ok) return true;
    if ((spin & 63) == 63) {
      const uint64_t now = globaltimer();
      if (t0 == 0) t0 = now;
      else if (now - t0 > timeout_ns) return false;
    }
  }
}

template <int K, bool W16, bool SYS, bool SGD>
__global__ void __launch_bounds__(kThreads)
tm_exchange_ll2_kernel(const __grid_constant__ ExchangeArgs a) {
  constexpr int LPU = W16 ? 1 : 2;
  __shared__ uint32_t s_calls;
  const int lr = blockIdx.x / a.C;
  const int c = blockIdx.x - lr * a.C;
  const int r = a.rank0 + lr;
  uint32_t* const tail = a.flags[r] + (size_t)(kPhases * TM_MAX_RANKS + 1) * a.flag_stride;
  if (threadIdx.x == 0) {
    s_calls = __ldcg(tail + kTailCalls);
    __threadfence();
    if (atomicAdd(tail + kTailRetire, 1u) == (uint32_t)a.C - 1) {
      tail[kTailRetire] = 0;
      tail[kTailCalls] = __ldcg(tail + kTailCalls) + 1;
    }
  }
  __syncthreads();
  const uint32_t epoch = s_calls + 1;
  const int par = (int)(s_calls & 1u);
  stamp(a, kStampStart);
  const int64_t n = a.P, L = a.L;
  const int64_t lpg = a.stage_stride / (32 * (int64_t)a.k);  // lines per slot
  const int64_t stride = (int64_t)a.C * kThreads;
  const int64_t t = (int64_t)c * kThreads + threadIdx.x;
  float* const x = a.x[lr];
  uint32_t st = 0;
  bool late = false;
  // line address: region 0 = reduce-scatter, 1 = allgather
  auto line = [&](int j, int vq, int region, int slot, int64_t unit) -> char* {
    return reinterpret_cast<char*>(a.stage[j]) + (int64_t)(par * a.nvec_alloc + vq) * a.stage_stride +
           (((int64_t)region * a.k + slot) * lpg + unit * LPU) * 16;
  };
  // ---------------- A: push every assigned unit to its owner -----------------
  const int64_t nu = (n + 3) / 4;
  for (int64_t u = t; u < nu; u += stride) {
    const int64_t g = u * 4;
    const int s = (int)(g / L);
    const int64_t us = (g - (int64_t)s * L) / 4;  // unit within segment s
    float f[4], fv[4];
    if (g + 4 <= n) {
      const float4 t4 = ld16_f(x + g);
      f[0] = t4.x; f[1] = t4.y; f[2] = t4.z; f[3] = t4.w;
    } else {
#pragma unroll
      for (int q = 0; q < 4; ++q) f[q] = g + q < n ? x[g + q] : 0.0f;
    }
    if constexpr (SGD) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        fv[q] = g + q < n ? sgd_v1(a.v[lr][g + q], a.g[lr][g + q], a.lr, a.mu) : 0.0f;
        f[q] = g + q < n ? __fadd_rn(f[q], fv[q]) : 0.0f;
      }
      if (a.nvec == 1) {
#pragma unroll
        for (int q = 0; q < 4; ++q)
          if (g + q < n) a.v[lr][g + q] = fv[q];
      } else {
        st |= unit_status<W16, 4>(fv);
      }
    }
    st |= unit_status<W16, 4>(f);
    for (int vq = 0; vq < a.nvec; ++vq) {
      const float* src = (SGD && vq == 1) ? fv : f;
      uint32_t w[2 * LPU];
      if constexpr (W16) {
        w[0] = pack_rn16x2(src[0], src[1]);
        w[1] = pack_rn16x2(src[2], src[3]);
      } else {
#pragma unroll
        for (int q = 0; q < 4; ++q) w[q] = __float_as_uint(src[q]);
      }
      char* dst = line(s, vq, 0, r, us);
#pragma unroll
      for (int h = 0; h < LPU; ++h) st_ll(dst + h * 16, w[2 * h], w[2 * h + 1], epoch);
    }
  }
  // ---------------- B: reduce the own segment's units, push the averages ------
  const int64_t seg_n = max((int64_t)0, min(L, n - (int64_t)r * L));
  const int64_t nus = (seg_n + 3) / 4;
  for (int64_t v = t; v < nus && !late; v += stride) {
    for (int vq = 0; vq < a.nvec && !late; ++vq) {
      float sm[4], tt[4];
#pragma unroll
      for (int j = 0; j < K; ++j) {
        uint4 ln[LPU];
        if (!poll_lines<LPU>(line(r, vq, 0, j, v), epoch, ln, a.timeout_ns)) {
          late = true;
          break;
        }
        if constexpr (W16) {
          const float2 lo = unpack16x2(ln[0].x), hi = unpack16x2(ln[0].z);
          tt[0] = lo.x; tt[1] = lo.y; tt[2] = hi.x; tt[3] = hi.y;
        } else {
          tt[0] = __uint_as_float(ln[0].x); tt[1] = __uint_as_float(ln[0].z);
          tt[2] = __uint_as_float(ln[LPU - 1].x); tt[3] = __uint_as_float(ln[LPU - 1].z);
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) sm[q] = j == 0 ? tt[q] : __fadd_rn(sm[q], tt[q]);
      }
      if (late) break;
      if (!a.sum) {
#pragma unroll
        for (int q = 0; q < 4; ++q) sm[q] = div_k<K>(sm[q]);
      } else if (W16) {
#pragma unroll
        for (int q = 0; q < 4; ++q) st |= status_of(sm[q], true) & TM_BIT_OVERFLOW16;
      }
      uint32_t w[2 * LPU];
      if constexpr (W16) {
        w[0] = pack_rn16x2(sm[0], sm[1]);
        w[1] = pack_rn16x2(sm[2], sm[3]);
      } else {
#pragma unroll
        for (int q = 0; q < 4; ++q) w[q] = __float_as_uint(sm[q]);
      }
#pragma unroll
      for (int j = 0; j < K; ++j) {
        char* dst = line(j, vq, 1, r, v);
#pragma unroll
        for (int h = 0; h < LPU; ++h) st_ll(dst + h * 16, w[2 * h], w[2 * h + 1], epoch);
      }
    }
  }
  // ---------------- C: pull every assigned unit's average from its owner ------
  for (int64_t u = t; u < nu && !late; u += stride) {
    const int64_t g = u * 4;
    const int s = (int)(g / L);
    const int64_t us = (g - (int64_t)s * L) / 4;
    for (int vq = 0; vq < a.nvec; ++vq) {
      uint4 ln[LPU];
      if (!poll_lines<LPU>(line(r, vq, 1, s, us), epoch, ln, a.timeout_ns)) {
        late = true;
        break;
      }
      float f[4];
      if constexpr (W16) {
        const float2 lo = unpack16x2(ln[0].x), hi = unpack16x2(ln[0].z);
        f[0] = lo.x; f[1] = lo.y; f[2] = hi.x; f[3] = hi.y;
      } else {
        f[0] = __uint_as_float(ln[0].x); f[1] = __uint_as_float(ln[0].z);
        f[2] = __uint_as_float(ln[LPU - 1].x); f[3] = __uint_as_float(ln[LPU - 1].z);
      }
      float* dstx = vq ? a.v[lr] : x;
      if (g + 4 <= n) {
        st16_f(dstx + g, make_float4(f[0], f[1], f[2], f[3]));
      } else {
#pragma unroll
        for (int q = 0; q < 4; ++q)
          if (g + q < n) dstx[g + q] = f[q];
      }
    }
  }
  if (late) st |= TM_BIT_TIMEOUT;
  if (st) atomicOr(a.status, st);
  stamp(a, kStampCast);
  stamp(a, kStampReady);
  stamp(a, kStampReduce);
  stamp(a, kStampReduced);
  stamp(a, kStampEnd);
}

template <int K, bool W16, bool SGD>
const void* exchange_fn(bool sys, int fl) {
  if (fl == kStagedTma)
    return sys ? reinterpret_cast<const void*>(&tm_exchange_tma_kernel<K, W16, true, SGD>)
               : reinterpret_cast<const void*>(&tm_exchange_tma_kernel<K, W16, false, SGD>);
  if (fl == kStagedWs)
    return sys ? reinterpret_cast<const void*>(&tm_exchange_ws_kernel<K, W16, true, SGD>)
               : reinterpret_cast<const void*>(&tm_exchange_ws_kernel<K, W16, false, SGD>);
  if (fl == kStagedTmaWs)
    return sys ? reinterpret_cast<const void*>(&tm_exchange_tmaws_kernel<K, W16, true, SGD>)
               : reinterpret_cast<const void*>(&tm_exchange_tmaws_kernel<K, W16, false, SGD>);
  if (fl == kStagedOneShot)
    return sys ? reinterpret_cast<const void*>(&tm_exchange_oneshot_kernel<K, W16, true, SGD>)
               : reinterpret_cast<const void*>(&tm_exchange_oneshot_kernel<K, W16, false, SGD>);
  if (fl == kStagedLL)
    return sys ? reinterpret_cast<const void*>(&tm_exchange_ll_kernel<K, W16, true, SGD>)
               : reinterpret_cast<const void*>(&tm_exchange_ll_kernel<K, W16, false, SGD>);
  if (fl == kStagedLL2)
    return sys ? reinterpret_cast<const void*>(&tm_exchange_ll2_kernel<K, W16, true, SGD>)
               : reinterpret_cast<const void*>(&tm_exchange_ll2_kernel<K, W16, false, SGD>);
  return sys ? reinterpret_cast<const void*>(&tm_exchange_kernel<K, W16, true, SGD>)
             : reinterpret_cast<const void*>(&tm_exchange_kernel<K, W16, false, SGD>);
}

// Kernel of k ranks, wire type, flag scope and flavour (SGD: the fused BSP step).
template <bool SGD>
const void* pick_exchange(int k, bool w16, bool sys, int fl) {
  switch (k) {
    case 2: return w16 ? exchange_fn<2, true, SGD>(sys, fl) : exchange_fn<2, false, SGD>(sys, fl);
    case 3: return w16 ? exchange_fn<3, true, SGD>(sys, fl) : exchange_fn<3, false, SGD>(sys, fl);
    case 4: return w16 ? exchange_fn<4, true, SGD>(sys, fl) : exchange_fn<4, false, SGD>(sys, fl);
    case 5: return w16 ? exchange_fn<5, true, SGD>(sys, fl) : exchange_fn<5, false, SGD>(sys, fl);
    case 6: return w16 ? exchange_fn<6, true, SGD>(sys, fl) : exchange_fn<6, false, SGD>(sys, fl);
    case 7: return w16 ? exchange_fn<7, true, SGD>(sys, fl) : exchange_fn<7, false, SGD>(sys, fl);
    case 8: return w16 ? exchange_fn<8, true, SGD>(sys, fl) : exchange_fn<8, false, SGD>(sys, fl);
    default: return nullptr;
  }
}

bool uses_tma(int fl) { return fl == kStagedTma || fl == kStagedTmaWs; }
int flavour_threads(int fl) { return uses_tma(fl) ? kTmaThreads : (fl == kStagedWs ? kWsThreads : kThreads); }

constexpr int kTmaSmem = (kInSlots + kOutSlots) * kSlotBytes;
static_assert(2 * CastGrp::kNin * CastGrp::kInB + RedGrp::kNin * RedGrp::kInB +
                  RedGrp::kNout * RedGrp::kOutB <= kTmaSmem, "tmaws phase-1 rings");
int flavour_smem(int fl) { return uses_tma(fl) ? kTmaSmem : 0; }

// Opt every TMA instantiation into its dynamic shared memory (idempotent).
cudaError_t prepare(const void* fn, int fl) {
  if (!uses_tma(fl)) return cudaSuccess;
  return cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, kTmaSmem);
}

}  // namespace
}  // namespace tmx
