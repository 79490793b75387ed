// Internal interface between the C++ runtime (tm_runtime.cpp) and the sm_100a
// kernels (tm_staged*.cu, tm_direct.cu, tm_bsp.cu, tm_easgd.cu,
// tm_loader_kernels.cu).  Not part of the public ABI.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "tm.h"

namespace tmx {

constexpr int kThreads = 256;       // threads per CTA of every kernel
constexpr int kVec = 8;             // elements per vector unit (16 B of fp16)
constexpr int64_t kAlign = 256;     // segment / chunk alignment in elements
constexpr int64_t kMinChunk = 2048; // smallest per-CTA chunk worth a barrier
// Tile-claim counter pairs per exchanger / per device (EASGD rounds): up to this
// many dynamic-tile launches may be in flight at once on different streams.
constexpr int kCtrSlots = 64;

// Flag pad of one rank: u32 flags[kPhases][TM_MAX_RANKS][C] followed by the
// per-CTA epoch counters u32 ctr[C] and a tail of kPadTail words; slot
// [phase][src][c] is written by rank `src` (remote store) and spun on by the
// owner of the pad; ctr[c] is private to CTA c of the owner.  Tail: [0] calls,
// [1] retire -- the one-shot kernel's per-rank call counter (the last CTA of a
// launch to retire increments `calls`, so every CTA of a launch reads the same
// value: the staging parity of the call) -- and [8 + src] the bootstrap
// self-check votes of rank src.
constexpr int kPhaseReady = 0;    // src finished its pre-cast of chunk c
constexpr int kPhaseReduced = 1;  // src finished summing its segment's chunk c
// The warp-specialised staged kernel splits a chunk into kWsSub sub-chunks with
// one READY phase each (0..kWsSub-1) and REDUCED = kWsSub.  The pad is laid out
// for kPhases phases; the per-CTA epoch counters follow them.
constexpr int kWsSub = 4;
constexpr int kPhases = kWsSub + 1;
constexpr int kPadTail = 16;
constexpr int kTailCalls = 0, kTailRetire = 1, kTailVotes = 8;
// Sub-chunk length of the warp-specialised kernels: a chunk is split into at
// most kWsSub sub-chunks of at least kWsMinSub elements (fewer flag rounds for
// small chunks, where each round costs more than the overlap gains).
constexpr int64_t kWsMinSub = 8192;

struct ExchangeArgs {
  void* stage[TM_MAX_RANKS];      // rank j's staging (k*L wire elems), as mapped here
  void* avg[TM_MAX_RANKS];        // rank j's averaged segment (L wire elems)
  uint32_t* flags[TM_MAX_RANKS];  // rank j's flag pad
  float* x[TM_MAX_RANKS];         // user buffers of the LOCAL ranks (index r - rank0)
  uint32_t* status;               // sticky status word (local)
  int64_t P, L, Lc;               // params, segment length, per-CTA chunk length
  int32_t k, rank0, C;            // ranks, first local rank, CTAs per rank (this call)
  int32_t flag_stride;            // C the flag pad was laid out for (>= C)
  int32_t sum;                    // SUBGD: sum, no 1/k
  uint64_t timeout_ns;
  uint64_t* stamps;               // diagnostics: %globaltimer per CTA and phase, or null
  // Fused BSP step (tm_bsp_step on the staged path): when sgd != 0
  // the pre-cast source of local rank lr is w' = fl(x + v'), with
  // v' = fl(fl(mu*v) - fl(lr*g)) from v[lr], g[lr]; v' is written back, w' is
  // not (the allgather overwrites every element of x).  Full range only.
  float* v[TM_MAX_RANKS];
  const float* g[TM_MAX_RANKS];
  float lr, mu;
  int32_t sgd;
  // Allgather outside the kernel (TM_AG_CE / TM_AG_NCCL): the kernel returns
  // after the REDUCED barrier and skips a6.
  int32_t ag_external;
  // Vectors exchanged by this launch: 1, or 2 for the BSP step with momentum
  // exchange (sgd != 0): vector 0 is w' (into x), vector 1 is v' (into v), both
  // through the same barriers.  Vector q's wire staging starts q * stage_stride
  // bytes after stage[j] (the one-shot kernel adds its parity buffers after
  // those: buffer (parity * nvec_alloc + q)), its averaged segment q *
  // avg_stride bytes after avg[j].
  int32_t nvec, nvec_alloc;
  int64_t stage_stride, avg_stride;
};

// Persistent fused exchange: pre-cast -> ready barrier -> reduce-scatter pull with
// fused sum/scale/cast -> reduced barrier -> allgather pull with fused widen.
// wire16: fp16 wire (ASA16) else fp32 (ASA).  grid = nlocal * C, cooperative.
// Phase stamps (tm_set_phase_log): slot [blockIdx][kStamp*] of the staged kernels.
constexpr int kStampSlots = 8;
enum { kStampStart = 0, kStampCast = 1, kStampReady = 2, kStampReduce = 3, kStampReduced = 4,
       kStampEnd = 5 };
// Staged kernel flavours.
//   kStagedOneShot: one READY barrier per call; every rank pulls every rank's
//   whole staging and reduces ALL segments itself in rank order (bitwise the
//   same average, no reduce-scatter / allgather split, no REDUCED barrier);
//   staging double-buffered by call parity.  Small segments only: it moves
//   (k-1) P s bytes per rank over the links instead of 2 (k-1)/k P s.
//   kStagedLL: no barrier at all -- each thread pushes its unit's wire lines,
//   the call's epoch inside every 16-byte line, into every rank's receive
//   buffer and polls its own for the k ranks' lines (tm_exchange_ll_kernel).
//   Smallest exchanges only: (k-1) P s bytes per rank, at half payload density.
//   kStagedLL2: the two-shot version (tm_exchange_ll2_kernel): units pushed to
//   their owner, the owner's averages pushed to every rank -- the ASA split with
//   epoch-tagged lines instead of barriers; 2 (k-1)/k P 2s bytes per rank.
enum StagedKernel { kStagedReg = 0, kStagedTma = 1, kStagedWs = 2, kStagedTmaWs = 3, kStagedOneShot = 4,
                    kStagedLL = 5, kStagedLL2 = 6 };
// Elements per CTA of the LL kernel (one 4-element unit per thread).
constexpr int64_t kLLChunk = 4 * 256;
// Per-CTA chunk granularity of the one-shot kernel (each CTA reduces its chunk
// of all k segments, k times the work of a two-phase CTA per element).
constexpr int64_t kOneShotChunk = 512;
cudaError_t launch_exchange(const ExchangeArgs& a, int nlocal, bool wire16, int flavour, cudaStream_t s);

// Single-process group, one pass (the "direct" path): pull the k contributions
// of each element from the k buffers, fused rn16 (q16) / ascending-rank sum /
// (1/k) / rn16, push the result to all k buffers.  Also AR when all ranks are
// local (q16 = false).
// tile_ctr: two zero-initialised device words for dynamic tile claiming (the
// kernel's last CTA resets them: no memset node per launch), or null for the
// static tile assignment.
// max_ctas > 0: a CTA budget (bucketed exchanges beside compute kernels): the
// register kernel (no shared memory, so its CTAs can co-reside with a GEMM's)
// on at most max_ctas CTAs.
cudaError_t launch_direct(float* const* bufs, int k, int64_t P, bool q16, bool sum,
                          uint32_t* status, unsigned long long* tile_ctr, cudaStream_t s,
                          int max_ctas = 0);

// concurrent: 0 exclusive, 1 hardware float atomic (red.add), 2 CAS-loop IEEE add
cudaError_t launch_easgd(float* x, float* c, int64_t n, float alpha, int concurrent,
                         cudaStream_t s);
cudaError_t launch_easgd_round(float* const* w, int nw, const int32_t* order, int norder,
                               float* c, int64_t n, float alpha, cudaStream_t s);
// EASGD against a centre sharded by segment: shard[s] holds c[s*L, (s+1)*L).
struct ShardArgs {
  float* shard[TM_MAX_RANKS];
  uint32_t* locks[TM_MAX_RANKS];    // per-chunk spin locks of shard s (locked mode)
  uint32_t* tickets[TM_MAX_RANKS];  // per-chunk count of applied updates (locked mode)
  int32_t* order_log;               // test hook: [s*nchunk + q][log_stride] worker ids
  int32_t log_stride;
  int32_t worker_id;
  int32_t k;
  int64_t L, P;
  bool sys;
  uint32_t* status;
  uint64_t timeout_ns;
};
constexpr int64_t kLockChunk = 4096;  // elements per lock in locked EASGD
cudaError_t launch_easgd_sharded(float* x, const ShardArgs& sa, float alpha, int concurrent,
                                 cudaStream_t s);
// Locked mode: each (shard, chunk) is updated under a spin lock, so every
// worker's update of an element is one atomic read-modify-write of the centre
// (per-worker atomic exchange) in arrival order.
cudaError_t launch_easgd_locked(float* x, const ShardArgs& sa, float alpha, cudaStream_t s);
// One BSP iteration (tm_bsp.cu): momentum-SGD step + exchange of the weights
// (and velocities when mom) for a single-process group, fused in one pass.
struct BspBufs {
  float* w[TM_MAX_RANKS];
  float* v[TM_MAX_RANKS];
  const float* g[TM_MAX_RANKS];
  float lr, mu;
};
// tile_ctr: as for launch_direct (two self-resetting words); null selects the
// register kernel.
cudaError_t launch_bsp_direct(const BspBufs& bb, int k, int64_t P, bool q16, bool mom,
                              uint32_t* status, unsigned long long* tile_ctr, cudaStream_t s);
cudaError_t launch_sgd(float* w, float* v, const float* g, int64_t n, float lr, float mu,
                       cudaStream_t s);
// Alg. 1 preprocessing (tm_loader_kernels.cu): mean subtraction, crop, mirror.
cudaError_t launch_preprocess(const uint8_t* raw, const float* mean, const int32_t* crop, float* out,
                              int n, int c, int h, int w, int ch, int cw, cudaStream_t s);
cudaError_t launch_cast_rn16(const float* in, uint16_t* out, int64_t n, cudaStream_t s);

// After an external allgather into `gather` (k*L wire elements in segment
// order): x[i] = widen(gather[i]) for i < P (fp16 wire).
cudaError_t launch_widen16(const void* gather, float* x, int64_t P, cudaStream_t s);

// Max co-resident CTAs of the exchange kernel on `device` (occupancy * SMs).
int exchange_max_ctas(int device, bool wire16, int k, int flavour);

}  // namespace tmx
