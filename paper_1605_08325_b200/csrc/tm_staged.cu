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
  stamp(a, kStampCast);

  if (!rank_barrier<K, SYS>(a, kPhaseReady, r, c, epoch, &s_abort)) return;
  stamp(a, kStampReady);

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

template <int K, bool W16, bool SYS>
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
  float* __restrict__ x = a.x[lr];
  const int64_t P = a.P, L = a.L;
  const int64_t e0 = (int64_t)c * a.Lc;
  const int64_t e1 = min(e0 + a.Lc, L);
  const int64_t nel = e1 > e0 ? e1 - e0 : 0;
  const int64_t Ls = ((nel + kWsSub - 1) / kWsSub + 255) / 256 * 256;  // sub-chunk length
  char* const stage_r = reinterpret_cast<char*>(a.stage[r]);
  const int grp = threadIdx.x / kWsGroup;
  const int tg = threadIdx.x - grp * kWsGroup;
  uint32_t st = 0;

  if (grp == 0) {
    // ------------------------------------------------ casters: a2 per sub-chunk
    constexpr int G = K < 4 ? K : 4;
    for (int t = 0; t < kWsSub; ++t) {
      const int64_t s0e = e0 + (int64_t)t * Ls;
      const int64_t s1e = min(s0e + Ls, e1);
      const int nu = s1e > s0e ? (int)((s1e - s0e) / E) : 0;
      for (int v = tg; v < nu; v += kWsGroup) {
        const int64_t ev = s0e + (int64_t)v * E;
#pragma unroll
        for (int sb = 0; sb < K; sb += G) {
          float f[G][E];
#pragma unroll
          for (int u = 0; u < G; ++u) {
            if (sb + u < K) {
              const int64_t g = (int64_t)(sb + u) * L + ev;
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
            if (sb + u < K) {
              const int64_t g = (int64_t)(sb + u) * L + ev;
              st |= unit_status<W16, E>(f[u]);
              st16_cg(stage_r + g * WB, U::encode(f[u]));
            }
          }
        }
      }
      named_bar(1, kWsGroup);  // every caster's stage writes of sub-chunk t done
      if (tg < K)
        st_release<SYS>(a.flags[tg] + (size_t)(t * TM_MAX_RANKS + r) * a.flag_stride + c, epoch);
    }
  } else {
    // ------------------------------------------------ reducers: a4 per sub-chunk
    const char* src[K];
#pragma unroll
    for (int j = 0; j < K; ++j) src[j] = reinterpret_cast<const char*>(a.stage[j]);
    char* const avg_r = reinterpret_cast<char*>(a.avg[r]);
    for (int t = 0; t < kWsSub; ++t) {
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
      for (int v = tg; v < nu; v += kWsGroup) {
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

  // ---------------- a6: allgather pull with all 16 warps ----------------------
  const int nu32 = (int)(nel / E);
  for (int v = threadIdx.x; v < nu32; v += kWsThreads) {
    const int64_t ev = e0 + (int64_t)v * E;
    uint4 raw[K];
#pragma unroll
    for (int j = 0; j < K; ++j) raw[j] = ld16_cg(reinterpret_cast<const char*>(a.avg[j]) + ev * WB);
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

// Runs n_items through the rings.  issue(i, slot, bar) [thread 0] starts the
// bulk loads of item i and arms `bar` with their byte count; compute(i, in, out)
// [all threads] transforms; store(i, out) [thread 0] issues the bulk stores.
// `use` / `outn` continue across phases so slot parities stay consistent.
template <class IssueF, class ComputeF, class StoreF>
__device__ __forceinline__ void tile_pipeline(int n_items, uint32_t& use, uint32_t& outn,
                                              char* in_ring, char* out_ring, uint64_t* full,
                                              IssueF issue, ComputeF compute, StoreF store) {
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int i = 0; i < kInSlots && i < n_items; ++i) {
      const uint32_t slot = (use + i) % kInSlots;
      issue(i, in_ring + slot * kSlotBytes, &full[slot]);
    }
  }
  for (int i = 0; i < n_items; ++i) {
    const uint32_t u = use + i;
    const uint32_t slot = u % kInSlots;
    mbar_wait(&full[slot], (u / kInSlots) & 1);
    char* out = out_ring + (outn % kOutSlots) * kSlotBytes;
    compute(i, in_ring + slot * kSlotBytes, out);
    fence_proxy_async_smem();                      // generic smem writes -> bulk store
    if (tid == 0) bulk_wait_read<kOutSlots - 2>();  // out slot of item i+1 is free
    __syncthreads();                               // every thread is done with slot / out
    if (tid == 0) {
      store(i, out);
      bulk_commit();
      if (i + kInSlots < n_items) issue(i + kInSlots, in_ring + slot * kSlotBytes, &full[slot]);
    }
    ++outn;
  }
  use += n_items;
}

// Drain this CTA's bulk stores and order them before the generic-proxy release.
__device__ __forceinline__ void drain_bulk_stores() {
  if (threadIdx.x == 0) {
    bulk_wait_all<0>();
    fence_proxy_async_global();
  }
}

// ---- dynamic work + rank-level barriers (TMA-engine kernel) ----------------
// The TMA kernel does not tie work to CTA chunks: within a phase every CTA of a
// rank claims items (tiles) from a per-rank counter until none are left, so no
// slow SM holds the phase back, and the phase ends with a RANK-level barrier:
// each CTA, after draining its bulk stores, fences and counts itself done; the
// rank's last CTA resets the phase's counters and publishes the epoch into
// every rank's pad slot [phase][r][0]; all CTAs then wait for every rank's slot.
// The epoch is one counter per rank (pad word kRankEpoch), read by every CTA at
// the start and advanced by the last CTA at READY -- no CTA can get there before
// all of them have read it.
//   READY   resets the pre-cast and allgather claim counters,
//   REDUCED resets the reduce-scatter claim counter.
// Reuse across exchanges follows the same argument as the per-CTA protocol with
// "rank" in place of "CTA c of the rank".
enum { kRankEpoch = 0, kDoneReady = 1, kDoneReduced = 2, kClaimCast = 3, kClaimReduce = 4,
       kClaimGather = 5 };

template <bool SYS>
__device__ __forceinline__ void fence_scope_sys() {
  if constexpr (SYS) __threadfence_system();
  else __threadfence();
}

// Streams claimed items through the rings until claim() returns -1.  Slot item
// ids live in smem (published to the consumers by the mbarrier arrive).
template <class ClaimF, class IssueF, class ComputeF, class StoreF>
__device__ __forceinline__ void dyn_tile_pipeline(uint32_t& use, uint32_t& outn, char* in_ring,
                                                  char* out_ring, uint64_t* full, int* slot_item,
                                                  ClaimF claim, IssueF issue, ComputeF compute,
                                                  StoreF store) {
  const int tid = threadIdx.x;
  auto fill = [&](uint32_t u) {  // thread 0: claim an item for ring use u
    const uint32_t slot = u % kInSlots;
    const int it = claim();
    slot_item[slot] = it;
    if (it < 0) mbar_expect_tx(&full[slot], 0);
    else issue(it, in_ring + slot * kSlotBytes, &full[slot]);
  };
  if (tid == 0)
    for (int q = 0; q < kInSlots; ++q) fill(use + q);
  uint32_t q = 0;
  for (;; ++q) {
    const uint32_t u = use + q;
    const uint32_t slot = u % kInSlots;
    mbar_wait(&full[slot], (u / kInSlots) & 1);
    const int it = slot_item[slot];
    if (it < 0) break;  // claims are monotone: every later slot is empty too
    char* out = out_ring + (outn % kOutSlots) * kSlotBytes;
    compute(it, in_ring + slot * kSlotBytes, out);
    fence_proxy_async_smem();
    if (tid == 0) bulk_wait_read<kOutSlots - 2>();
    __syncthreads();
    if (tid == 0) {
      store(it, out);
      bulk_commit();
      fill(u + kInSlots);
    }
    ++outn;
  }
  // consume the remaining (empty, already completed) prefetched slots so every
  // slot's phase parity stays in step for the next phase
  for (uint32_t r = 1; r < kInSlots; ++r) {
    const uint32_t u = use + q + r;
    mbar_wait(&full[u % kInSlots], (u / kInSlots) & 1);
  }
  __syncthreads();  // nobody still reads slot_item before the next phase refills it
  use += q + kInSlots;
}

template <int K, bool SYS>
__device__ __forceinline__ bool rank_level_barrier(const ExchangeArgs& a, int phase, int r,
                                                   uint32_t* rk, uint32_t epoch, int done_idx,
                                                   int reset0, int reset1, int* s_abort) {
  __syncthreads();
  if (threadIdx.x == 0) {
    fence_scope_sys<SYS>();  // this CTA's writes (all threads, via bar.sync) before the count
    const uint32_t old = atomicAdd(rk + done_idx, 1u);
    if (old == (uint32_t)a.C - 1) {  // the rank's last CTA for this phase
      fence_scope_sys<SYS>();
      rk[done_idx] = 0;
      rk[reset0] = 0;
      if (reset1 >= 0) rk[reset1] = 0;
      if (phase == kPhaseReady) rk[kRankEpoch] = epoch;
      __threadfence();
      for (int j = 0; j < a.k; ++j)
        st_release<SYS>(a.flags[j] + (size_t)(phase * TM_MAX_RANKS + r) * a.flag_stride, epoch);
    }
  }
  if (threadIdx.x < K) {
    const uint32_t* mine = a.flags[r] + (size_t)(phase * TM_MAX_RANKS + threadIdx.x) * a.flag_stride;
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
__global__ void __launch_bounds__(kTmaThreads, 1)
tm_exchange_tma_kernel(const __grid_constant__ ExchangeArgs a) {
  using U = Unit<W16>;
  constexpr int E = U::kElems;      // elements per 16-byte wire unit
  constexpr int WB = W16 ? 2 : 4;   // wire bytes per element
  constexpr int TP = 8192;          // a2 tile: fp32 in 32 KB, wire out <= 32 KB
  // a4 tile: k sources of TR wire elements fit one 32 KB slot; a multiple of 256
  // elements keeps every source's smem offset and byte count 16-byte aligned.
  constexpr int TR_RAW = kSlotBytes / (K * WB) / 256 * 256;
  constexpr int TR = TR_RAW < 4096 ? TR_RAW : 4096;
  static_assert(TR >= 256, "a4 tile too small");
  constexpr int TA = 8192;          // a6 tile: wire in <= 32 KB, fp32 out 32 KB
  extern __shared__ __align__(128) unsigned char smem[];
  char* in_ring = reinterpret_cast<char*>(smem);
  char* out_ring = in_ring + kInSlots * kSlotBytes;
  __shared__ __align__(8) uint64_t full[kInSlots];
  __shared__ int slot_item[kInSlots];
  __shared__ int s_abort;
  __shared__ uint32_t s_epoch;

  const int lr = blockIdx.x / a.C;
  const int r = a.rank0 + lr;
  float* __restrict__ x = a.x[lr];
  const int64_t P = a.P, L = a.L, P4 = P & ~int64_t(3);
  char* const stage_r = reinterpret_cast<char*>(a.stage[r]);
  // rank-level words after the per-CTA counters of the pad
  uint32_t* const rk = a.flags[r] + (size_t)kPhases * TM_MAX_RANKS * a.flag_stride + a.flag_stride;
  const int tid = threadIdx.x;

  if (tid == 0) {
    s_abort = 0;
    s_epoch = *reinterpret_cast<volatile uint32_t*>(rk + kRankEpoch) + 1;
    for (int i = 0; i < kInSlots; ++i) mbar_init(&full[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const uint32_t epoch = s_epoch;
  stamp(a, kStampStart);
  uint32_t use = 0, outn = 0, st = 0;
  auto claimer = [&](int idx, int limit) {
    return [=]() -> int {
      const int t = (int)atomicAdd(rk + idx, 1u);
      return t < limit ? t : -1;
    };
  };

  // ---------------- a2: pre-cast x -> own stage (every segment, tile by tile) --
  {
    const int nt = (int)((L + TP - 1) / TP);  // tiles per segment
    auto geom = [&](int i, int64_t& g0, int64_t& n) {
      const int sg = i / nt, t = i - sg * nt;
      g0 = (int64_t)sg * L + (int64_t)t * TP;
      n = min((int64_t)TP, L - (int64_t)t * TP);
    };
    dyn_tile_pipeline(
        use, outn, in_ring, out_ring, full, slot_item, claimer(kClaimCast, K * nt),
        [&](int i, char* slot, uint64_t* bar) {
          int64_t g0, n;
          geom(i, g0, n);
          const int64_t nb = max((int64_t)0, min(g0 + n, P4) - g0);  // bulk-loadable elements
          mbar_expect_tx(bar, (uint32_t)(nb * 4));
          if (nb > 0) bulk_load(slot, x + g0, (uint32_t)(nb * 4), bar);
        },
        [&](int i, const char* in, char* out) {
          int64_t g0, n;
          geom(i, g0, n);
          const int nbi = (int)max((int64_t)0, min(g0 + n, P4) - g0);
          const float* fin = reinterpret_cast<const float*>(in);
          for (int v = tid; v < (int)(n / E); v += kTmaThreads) {
            float f[E];
            if ((v + 1) * E <= nbi) {
#pragma unroll
              for (int q = 0; q < E; q += 4) {
                const float4 t4 = reinterpret_cast<const float4*>(fin + v * E)[q / 4];
                f[q] = t4.x; f[q + 1] = t4.y; f[q + 2] = t4.z; f[q + 3] = t4.w;
              }
            } else {
#pragma unroll
              for (int q = 0; q < E; ++q) {
                const int e = v * E + q;
                f[q] = e < nbi ? fin[e] : (g0 + e < P ? x[g0 + e] : 0.0f);
              }
            }
            st |= unit_status<W16, E>(f);
            reinterpret_cast<uint4*>(out)[v] = U::encode(f);
          }
        },
        [&](int i, const char* out) {
          int64_t g0, n;
          geom(i, g0, n);
          bulk_store(stage_r + g0 * WB, out, (uint32_t)(n * WB));
        });
  }
  if (st) atomicOr(a.status, st);
  drain_bulk_stores();
  stamp(a, kStampCast);
  if (!rank_level_barrier<K, SYS>(a, kPhaseReady, r, rk, epoch, kDoneReady, kClaimCast, kClaimGather,
                                  &s_abort))
    return;
  stamp(a, kStampReady);
  if (tid == 0) fence_proxy_async_global();  // peers' staging, acquired above -> bulk loads

  // ---------------- a4: reduce-scatter pull (TMA from every rank's stage) ----
  {
    char* const avg_r = reinterpret_cast<char*>(a.avg[r]);
    const int nt = (int)((L + TR - 1) / TR);
    dyn_tile_pipeline(
        use, outn, in_ring, out_ring, full, slot_item, claimer(kClaimReduce, nt),
        [&](int i, char* slot, uint64_t* bar) {
          const int64_t e = (int64_t)i * TR;
          const int64_t n = min((int64_t)TR, L - e);
          mbar_expect_tx(bar, (uint32_t)(K * n * WB));
#pragma unroll
          for (int j = 0; j < K; ++j)
            bulk_load(slot + j * TR * WB, reinterpret_cast<const char*>(a.stage[j]) + ((int64_t)r * L + e) * WB,
                      (uint32_t)(n * WB), bar);
        },
        [&](int i, const char* in, char* out) {
          const int64_t e = (int64_t)i * TR;
          const int n = (int)min((int64_t)TR, L - e);
          for (int v = tid; v < n / E; v += kTmaThreads) {
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
          const int64_t e = (int64_t)i * TR;
          const int64_t n = min((int64_t)TR, L - e);
          bulk_store(avg_r + e * WB, out, (uint32_t)(n * WB));
        });
  }
  if (st) atomicOr(a.status, st);
  drain_bulk_stores();
  stamp(a, kStampReduce);
  if (!rank_level_barrier<K, SYS>(a, kPhaseReduced, r, rk, epoch, kDoneReduced, kClaimReduce, -1,
                                  &s_abort))
    return;
  stamp(a, kStampReduced);
  if (tid == 0) fence_proxy_async_global();

  // ---------------- a6: allgather pull (TMA from every rank's avg) ----------
  {
    const int nt = (int)((L + TA - 1) / TA);
    auto geom = [&](int i, int& j, int64_t& e, int64_t& n) {
      j = i / nt;
      const int t = i - j * nt;
      e = (int64_t)t * TA;
      n = min((int64_t)TA, L - e);
    };
    dyn_tile_pipeline(
        use, outn, in_ring, out_ring, full, slot_item, claimer(kClaimGather, K * nt),
        [&](int i, char* slot, uint64_t* bar) {
          int j;
          int64_t e, n;
          geom(i, j, e, n);
          mbar_expect_tx(bar, (uint32_t)(n * WB));
          bulk_load(slot, reinterpret_cast<const char*>(a.avg[j]) + e * WB, (uint32_t)(n * WB), bar);
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
          for (int v = tid; v < (int)(n / E); v += kTmaThreads) {
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
        });
  }
  if (tid == 0) bulk_wait_all<0>();  // kernel exit also waits; explicit for clarity
  stamp(a, kStampEnd);
}

template <int K, bool W16>
const void* exchange_fn(bool sys, int fl) {
  if (fl == kStagedTma)
    return sys ? reinterpret_cast<const void*>(&tm_exchange_tma_kernel<K, W16, true>)
               : reinterpret_cast<const void*>(&tm_exchange_tma_kernel<K, W16, false>);
  if (fl == kStagedWs)
    return sys ? reinterpret_cast<const void*>(&tm_exchange_ws_kernel<K, W16, true>)
               : reinterpret_cast<const void*>(&tm_exchange_ws_kernel<K, W16, false>);
  return sys ? reinterpret_cast<const void*>(&tm_exchange_kernel<K, W16, true>)
             : reinterpret_cast<const void*>(&tm_exchange_kernel<K, W16, false>);
}

const void* pick_exchange(int k, bool w16, bool sys, int fl) {
  switch (k) {
    case 2: return w16 ? exchange_fn<2, true>(sys, fl) : exchange_fn<2, false>(sys, fl);
    case 3: return w16 ? exchange_fn<3, true>(sys, fl) : exchange_fn<3, false>(sys, fl);
    case 4: return w16 ? exchange_fn<4, true>(sys, fl) : exchange_fn<4, false>(sys, fl);
    case 5: return w16 ? exchange_fn<5, true>(sys, fl) : exchange_fn<5, false>(sys, fl);
    case 6: return w16 ? exchange_fn<6, true>(sys, fl) : exchange_fn<6, false>(sys, fl);
    case 7: return w16 ? exchange_fn<7, true>(sys, fl) : exchange_fn<7, false>(sys, fl);
    case 8: return w16 ? exchange_fn<8, true>(sys, fl) : exchange_fn<8, false>(sys, fl);
    default: return nullptr;
  }
}

int flavour_threads(int fl) { return fl == kStagedTma ? kTmaThreads : (fl == kStagedWs ? kWsThreads : kThreads); }

constexpr int kTmaSmem = (kInSlots + kOutSlots) * kSlotBytes;

// Opt every TMA instantiation into its dynamic shared memory (idempotent).
cudaError_t prepare(const void* fn, int fl) {
  if (fl != kStagedTma) return cudaSuccess;
  return cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, kTmaSmem);
}

}  // namespace

int exchange_max_ctas(int device, bool wire16, int k, int fl) {
  const void* fn = pick_exchange(k, wire16, true, fl);
  if (!fn) return 0;
  if (prepare(fn, fl) != cudaSuccess) return 0;
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, flavour_threads(fl),
                                                    fl == kStagedTma ? kTmaSmem : 0) != cudaSuccess)
    return 0;
  return per_sm * sm_count(device);
}

cudaError_t launch_exchange(const ExchangeArgs& a, int nlocal, bool wire16, int fl, cudaStream_t s) {
  // System-scope flags only when some peer rank lives in another process
  // (another GPU, over NVLink); a single-process group syncs at GPU scope.
  const void* fn = pick_exchange(a.k, wire16, nlocal != a.k, fl);
  if (!fn) return cudaErrorInvalidValue;
  cudaError_t e = prepare(fn, fl);
  if (e != cudaSuccess) return e;
  void* params[] = {const_cast<ExchangeArgs*>(&a)};
  // Cooperative launch: guarantees every CTA is co-resident, which the
  // per-CTA flag barriers need when several ranks share this device.
  return cudaLaunchCooperativeKernel(fn, dim3(nlocal * a.C), dim3(flavour_threads(fl)), params,
                                     fl == kStagedTma ? kTmaSmem : 0, s);
}

}  // namespace tmx
