// C++ runtime behind include/tm.h: the process-global exchanger context, the
// segmented layout, library-owned device memory, CUDA IPC
// peer mappings (the NVLink/NVSwitch data plane), the NCCL communicator used by
// AR across processes (dlopen'ed: the same libnccl.so.2 torch already loaded),
// argument validation and the sticky status word.
//
// PAPER.md L94-106 / L613-614: the paper ran one MPI process per GPU with
// CUDA-aware OpenMPI.  Here one process per GPU is kept, but MPI is replaced by
// (i) a one-time bootstrap in which the processes swap IPC handles (moved by
// the caller, e.g. torch.distributed all_gather_object) and (ii) in-kernel
// loads from peer memory with flag synchronisation.

#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>
#include <nvtx3/nvToolsExt.h>  // header-only; ranges are no-ops unless a tool (nsys) is attached
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

#include <algorithm>
#include <chrono>
#include <mutex>
#include <numeric>
#include <vector>

#include "tm.h"
#include "tm_internal.h"

namespace {

using tmx::ExchangeArgs;

// Host-side NVTX range around each enqueueing call (the exchange
// appears as a named range on nsys timelines next to its kernels).
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

constexpr uint32_t kMagic = 0x544d4558u;  // "TMEX"
constexpr uint32_t kVersion = 3;
constexpr uint64_t kDefaultTimeoutNs = 10ull * 1000 * 1000 * 1000;

struct Blob {
  uint32_t magic, version;
  int32_t rank0, nlocal, size, strategy, C, pid;
  int64_t P, L, Lc, rank_stride;
  int64_t off_stage, off_avg, off_flags, off_center;
  int32_t has_nccl, device_ordinal;
  int32_t ag_nccl;  // TM_ALLGATHER=nccl at init: every rank must agree (a collective)
  // Staged kernel flavour and allgather mode chosen at init (TM_STAGED_KERNEL /
  // TM_ALLGATHER can differ per process): the flavours use different flag phases
  // (READY_0..3 + REDUCED = 4 for the warp-specialised ones, READY = 0 and
  // REDUCED = 1 for the others), so ranks running different flavours would read
  // each other's READY_1 as REDUCED.  Every rank must agree.
  int32_t staged_kernel, ag_mode;
  cudaIpcMemHandle_t handle;
  ncclUniqueId nccl_id;
};
static_assert(sizeof(Blob) <= TM_BLOB_BYTES, "blob too large");

// --- NCCL, resolved at run time -------------------------------------------
struct Nccl {
  void* lib = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  bool load() {
    if (lib) return true;
    const char* path = getenv("TM_NCCL_LIB");
    lib = dlopen(path && *path ? path : "libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!lib) return false;
    GetUniqueId = (decltype(GetUniqueId))dlsym(lib, "ncclGetUniqueId");
    CommInitRank = (decltype(CommInitRank))dlsym(lib, "ncclCommInitRank");
    AllReduce = (decltype(AllReduce))dlsym(lib, "ncclAllReduce");
    CommDestroy = (decltype(CommDestroy))dlsym(lib, "ncclCommDestroy");
    AllGather = (decltype(AllGather))dlsym(lib, "ncclAllGather");
    return GetUniqueId && CommInitRank && AllReduce && CommDestroy && AllGather;
  }
};

struct Ctx {
  bool inited = false, ready = false;
  int64_t P = 0, L = 0, Lc = 0;
  int k = 0, rank0 = 0, nlocal = 0, device = 0, strategy = 0, C = 0;
  int flag_c = 0;  // CTA stride of the flag pad, fixed at init (C may shrink on a self-check fallback)
  int nprocs = 1, proc = 0;
  int64_t rank_stride = 0, off_stage = 0, off_avg = 0, off_flags = 0, off_center = 0;
  int64_t stage_stride = 0, avg_stride = 0;  // bytes between staging / avg buffers (vectors, parities)
  int nvec_alloc = 2;                        // staging buffers per parity (w and v of a BSP step)
  int selfcheck = 0;                         // bootstrap known-answer check: 0 not run, 1 passed, 2 fell back
  int64_t off_locks = 0, off_tickets = 0;  // EASGD locked mode
  int32_t* order_log = nullptr;            // test hook (tm_easgd_set_order_log)
  uint64_t* stamps = nullptr;              // diagnostics (tm_set_phase_log)
  int64_t stamps_cap = 0;
  int order_log_stride = 0;
  int64_t slab_bytes = 0;
  char* slab = nullptr;
  uint32_t* status = nullptr;
  char* peer_base[TM_MAX_RANKS] = {};  // per process (only the opened ones)
  char* rank_base[TM_MAX_RANKS] = {};  // per global rank, as mapped on this device
  uint32_t epoch = 0;
  // Tile-claim counters of the dynamic-tile kernels (direct, BSP): a ring of
  // kCtrSlots (claim, retire) pairs after the status word; each launch takes the
  // next slot, so launches running concurrently on different streams never share
  // a counter (a kernel resets its pair when its last CTA retires).
  unsigned long long* tile_ctrs = nullptr;
  uint32_t ctr_seq = 0;
  int range_ctas = 0;  // CTA budget of range (bucket) exchanges per rank; 0 = none
  int path = TM_PATH_AUTO;
  int staged_kernel = tmx::kStagedTma;  // staged kernel flavour, fixed at init (it sets C)
  int ag_mode = TM_AG_SM;               // tm_allgather of the staged path
  bool want_nccl_ag = false;            // TM_ALLGATHER=nccl at init: build a communicator
  bool sum = false;  // TM_OP_SUM (SUBGD)
  uint64_t timeout_ns = kDefaultTimeoutNs;
  ncclComm_t comm = nullptr;
  ncclUniqueId nccl_id{};
  bool have_nccl_id = false;
};

Ctx g;
Nccl g_nccl;
std::mutex g_mu;

// Flavour thresholds by segment length L (elements per rank) and k, from the r02
// latency tables (profiles/r02/latency/, k processes concurrent under MPS and k
// ranks in one process): the one-shot kernel moves (k-1) P s bytes per rank
// instead of 2 (k-1)/k P s -- the same at k = 2, where its single barrier wins
// at every measured size (two processes under MPS: P = 2 Ki .. 2 Mi, and up to
// AlexNet's 346.6 vs 367.6 us for tma) -- so at k > 2 it pays only while the
// call is latency-bound: up to L = 32 Ki at k <= 4 (11.4 vs 15.2 us for the
// register kernel at P = 64 Ki), 16 Ki at k = 8 (19.5 vs 20.8 us at P = 128 Ki;
// 25.5 vs 22.3 us at 256 Ki).  At k = 2 the cap is L = 1 Mi all the same: over
// NVLink the one-shot's pull cannot start on a chunk before that chunk's whole
// pre-cast, while the warp-specialised two-phase kernel overlaps the pre-cast
// (HBM) with the pull (NVLink) sub-chunk by sub-chunk -- an overlap one GPU,
// where both are HBM traffic, cannot show; above ~2 M parameters the pre-cast
// (6P bytes of HBM) is long enough for that to matter.
// The register two-phase kernel up to L = 32 Ki, the TMA-engine kernels above.
int64_t oneshot_max_l(int k) { return k == 2 ? (int64_t)1 << 20 : k <= 4 ? 32768 : 16384; }
// The LL kernel (no barrier; the epoch travels inside every wire line) below
// these segment lengths, from the r02 LL latency tables (profiles/r02/ll/: k
// processes concurrent under MPS, and k ranks in one process; 64 exchanges per
// graph).  Under MPS, LL vs the previous default: k = 2 4.6-5.5 us vs 7.5-17 us
// up to P = 256 Ki and 10.4 vs 18.9 us at 1 Mi; k = 4 5.3-9.8 vs 8.5-19.5 us up
// to 256 Ki, 17.6 vs 23.3 at 512 Ki, 45.1 vs 26.0 at 1 Mi; k = 8 7.3-9.5 vs
// 9.8-13.7 us up to 64 Ki, level at 128 Ki, behind above (every rank pushes
// every element to every rank, and polls k lines per unit).  Above LL, the
// two-shot LL2 kernel (profiles/r02/ll2/): under MPS k = 4 12.4 vs 18.3 us (LL)
// at P = 512 Ki, 21.0 vs 25.6 (tma) at 1 Mi; k = 8 15.5 vs 16.2 (one-shot) at
// 128 Ki, 19.0 vs 21.9 (reg) at 256 Ki, 27.5 vs 27.7 (one-shot) at 512 Ki (one
// process: 9.9 / 13.5 / 20.4 vs 12.8 / 14.1 / 22.7); k = 2 19.0 vs 21.3
// (one-shot) at 2 Mi.  So LL up to P = 1 Mi at k = 2, 256 Ki at k <= 4, 64 Ki
// above; LL2 up to 2 Mi, 1 Mi and 512 Ki; the two-phase kernels above.
int64_t ll_max_l(int k) { return k == 2 ? (int64_t)1 << 19 : k <= 4 ? (int64_t)1 << 16 : 8192; }
int64_t ll2_max_l(int k) { return k == 2 ? (int64_t)1 << 20 : k <= 4 ? (int64_t)1 << 18 : (int64_t)1 << 16; }
constexpr int64_t kRegMaxL = 32768;

int64_t env_i64(const char* name, int64_t dflt) {
  const char* v = getenv(name);
  return (v && *v) ? atoll(v) : dflt;
}

// Per-CTA chunk of the one-shot kernel (TM_ONESHOT_CHUNK, a multiple of 256,
// overrides for A/B runs; every rank must use the same value).
int64_t oneshot_chunk() {
  const int64_t c = env_i64("TM_ONESHOT_CHUNK", tmx::kOneShotChunk);
  return c >= 256 ? c / 256 * 256 : tmx::kOneShotChunk;
}

// The allgather decision step (north star: "falling back to NCCL allgather ...
// only where it measures faster"): TM_AG_TABLE names a table measured on the
// multi-GPU box (tools/ag_decide.py writes it from tools/multigpu_eval.sh's
// bench lines), one rule per line "k L_max mode" (mode sm | ce | nccl, '#'
// comments); the first rule with this k and L <= L_max picks the mode.  No
// table or no matching rule: the fused SM pull (measured fastest on one GPU:
// 0.97 vs 1.85 ms for the copy engines, profiles/r01/allgather_modes.jsonl).
// Every rank reads the same table, and the bootstrap checks the modes agree.
const char* ag_table_mode(const char* path, int k, int64_t L) {
  FILE* f = fopen(path, "r");
  if (!f) return nullptr;
  char line[256];
  const char* mode = nullptr;
  while (!mode && fgets(line, sizeof line, f)) {
    int kk = 0;
    long long lmax = 0;
    char m[16] = {0};
    if (line[0] == '#' || sscanf(line, "%d %lld %15s", &kk, &lmax, m) != 3) continue;
    if (kk != k || L > lmax) continue;
    mode = !strcmp(m, "nccl") ? "nccl" : !strcmp(m, "ce") ? "ce" : "sm";
  }
  fclose(f);
  return mode;
}

bool wire16(int strategy) { return strategy == TM_ASA16; }
int wire_bytes(int strategy) { return wire16(strategy) ? 2 : 4; }
int64_t round_up(int64_t a, int64_t b) { return (a + b - 1) / b * b; }

void debug_cuda(const char* where, cudaError_t e) {
  if (getenv("TM_DEBUG")) fprintf(stderr, "[tm] %s: %s\n", where, cudaGetErrorString(e));
}

int cuda_fail(const char* where, cudaError_t e) {
  debug_cuda(where, e);
  return TM_E_CUDA;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

void fill_rank_bases_local() {
  for (int i = 0; i < g.nlocal; ++i) g.rank_base[g.rank0 + i] = g.slab + (int64_t)i * g.rank_stride;
}

void release() {
  if (g.comm && g_nccl.CommDestroy) g_nccl.CommDestroy(g.comm);
  g.comm = nullptr;
  for (int p = 0; p < TM_MAX_RANKS; ++p) {
    if (g.peer_base[p]) cudaIpcCloseMemHandle(g.peer_base[p]);
    g.peer_base[p] = nullptr;
  }
  if (g.slab) cudaFree(g.slab);
  g = Ctx();
}

// The next launch's tile-claim counter pair (see Ctx::tile_ctrs).
unsigned long long* next_tile_ctr() {
  return g.tile_ctrs + 2 * (size_t)(g.ctr_seq++ % tmx::kCtrSlots);
}

// Launch arguments for an exchange of elements [off, off + n) of the callers'
// buffers.  The range gets a segmented layout of its own (a1): L' =
// roundup(ceil(n/k), 256) <= L, so it fits the staging allocated for P; C' <= C
// CTAs per rank, and the flag pad keeps the stride C it was laid out with.
ExchangeArgs make_args(float* const* bufs, int64_t off, int64_t n) {
  ExchangeArgs a{};
  for (int j = 0; j < g.k; ++j) {
    a.stage[j] = g.rank_base[j] + g.off_stage;
    a.avg[j] = g.rank_base[j] + g.off_avg;
    a.flags[j] = reinterpret_cast<uint32_t*>(g.rank_base[j] + g.off_flags);
  }
  for (int i = 0; i < g.nlocal; ++i) a.x[i] = bufs[i] + off;
  a.status = g.status;
  a.P = n;
  if (off == 0 && n == g.P) {
    a.L = g.L;
    a.Lc = g.Lc;
    a.C = g.C;
  } else {
    a.L = round_up((n + g.k - 1) / g.k, tmx::kAlign);
    const int64_t chunk = g.staged_kernel == tmx::kStagedOneShot ? oneshot_chunk() : tmx::kMinChunk;
    // the LL kernel spreads the call's n elements (not a segment) over its CTAs
    const bool ll = g.staged_kernel == tmx::kStagedLL || g.staged_kernel == tmx::kStagedLL2;
    const int64_t want = ll ? std::max<int64_t>(1, (n + tmx::kLLChunk - 1) / tmx::kLLChunk)
                            : std::max<int64_t>(1, (a.L + chunk - 1) / chunk);
    a.C = (int)std::min<int64_t>(g.C, want);
    if (g.range_ctas > 0) a.C = std::min(a.C, g.range_ctas);  // bucket beside compute kernels
    a.Lc = round_up((a.L + a.C - 1) / a.C, tmx::kAlign);
  }
  a.nvec = 1;
  a.nvec_alloc = g.nvec_alloc;
  a.stage_stride = g.stage_stride;
  a.avg_stride = g.avg_stride;
  a.flag_stride = g.flag_c;
  a.k = g.k;
  a.rank0 = g.rank0;
  a.sum = g.sum ? 1 : 0;
  a.timeout_ns = g.timeout_ns;
  a.stamps = (g.stamps && g.stamps_cap >= (int64_t)g.nlocal * a.C * tmx::kStampSlots) ? g.stamps : nullptr;
  return a;
}

// a6 outside the kernel (TM_AG_CE / TM_AG_NCCL), after the kernel's REDUCED
// barrier: gather the k averaged segments (a.L wire elements each) of every local
// rank into its own staging (free: every rank has finished its reduce-scatter
// reads of it), then widen into the caller's buffer.  ASA on the copy engines
// copies straight into the caller's buffer (no widening).  Reuse: the next
// exchange overwrites staging (pre-cast) and avg (reduce-scatter, after READY
// from every rank) only after this stream-ordered work, and NCCL has consumed
// its send buffer when its kernel completes.
int external_allgather(const ExchangeArgs& a, cudaStream_t s) {
  const int wb = wire_bytes(g.strategy);
  for (int vq = 0; vq < a.nvec; ++vq)
  for (int i = 0; i < g.nlocal; ++i) {
    const int r = g.rank0 + i;
    char* gather = static_cast<char*>(a.stage[r]) + vq * a.stage_stride;  // vector vq's own staging
    float* x = vq ? a.v[i] : a.x[i];
    const char* avg_r = static_cast<const char*>(a.avg[r]) + vq * a.avg_stride;
    if (g.ag_mode == TM_AG_NCCL) {
      if (!g.comm) return TM_E_NCCL;
      ncclResult_t nr = g_nccl.AllGather(avg_r, gather, (size_t)a.L,
                                         wb == 2 ? ncclFloat16 : ncclFloat32, g.comm, s);
      if (nr != ncclSuccess) return TM_E_NCCL;
    }
    for (int j = 0; j < g.k; ++j) {
      const int64_t n = std::min(a.L, a.P - (int64_t)j * a.L);  // elements of segment j < P
      const char* avg_j = static_cast<const char*>(a.avg[j]) + vq * a.avg_stride;
      if (g.ag_mode == TM_AG_CE) {
        cudaError_t e;
        if (wb == 4) {
          if (n <= 0) break;
          e = cudaMemcpyAsync(x + (int64_t)j * a.L, avg_j, (size_t)n * 4, cudaMemcpyDefault, s);
        } else {
          e = cudaMemcpyAsync(gather + (int64_t)j * a.L * wb, avg_j, (size_t)a.L * wb,
                              cudaMemcpyDefault, s);
        }
        if (e != cudaSuccess) return cuda_fail("allgather copy", e);
      } else if (wb == 4 && n > 0) {  // NCCL, fp32: segment j of the gather -> caller
        cudaError_t e = cudaMemcpyAsync(x + (int64_t)j * a.L, gather + (int64_t)j * a.L * wb,
                                        (size_t)n * 4, cudaMemcpyDeviceToDevice, s);
        if (e != cudaSuccess) return cuda_fail("allgather copy", e);
      }
    }
    if (wb == 2) {
      cudaError_t e = tmx::launch_widen16(gather, x, a.P, s);
      if (e != cudaSuccess) return cuda_fail("launch_widen16", e);
    }
  }
  return TM_OK;
}

int launch_staged(ExchangeArgs& a, cudaStream_t s) {
  // the one-shot kernel has no allgather phase to hand to the copy engines / NCCL
  a.ag_external = g.ag_mode != TM_AG_SM && g.staged_kernel != tmx::kStagedOneShot &&
                  g.staged_kernel != tmx::kStagedLL && g.staged_kernel != tmx::kStagedLL2;
  cudaError_t e = tmx::launch_exchange(a, g.nlocal, wire16(g.strategy), g.staged_kernel, s);
  if (e != cudaSuccess) return cuda_fail("launch_exchange", e);
  ++g.epoch;  // host-side count for tm_layout; the kernels keep their own
  return a.ag_external ? external_allgather(a, s) : TM_OK;
}

int effective_path() {
  if (g.path != TM_PATH_AUTO) return g.path;
  return g.nlocal == g.k ? TM_PATH_DIRECT : TM_PATH_STAGED;
}

int do_exchange(float* const* bufs, int nbufs, int64_t off, int64_t n, cudaStream_t s) {
  if (!g.inited || !g.ready || g.strategy == TM_EASGD) return TM_E_STATE;
  if (nbufs != g.nlocal || !bufs) return TM_E_ARG;
  if (off < 0 || n < 0 || off + n > g.P) return TM_E_ARG;
  if (off % 4) return TM_E_ALIGN;
  for (int i = 0; i < nbufs; ++i) {
    if (!bufs[i]) return TM_E_ARG;
    if (!aligned16(bufs[i])) return TM_E_ALIGN;
  }
  if (g.k == 1 || n == 0) return TM_OK;  // reading Q10: identity, nothing launched
  cudaSetDevice(g.device);
  if (g.nlocal == g.k && (g.strategy == TM_AR || effective_path() == TM_PATH_DIRECT)) {
    float* shifted[TM_MAX_RANKS];
    for (int i = 0; i < nbufs; ++i) shifted[i] = bufs[i] + off;
    const char* st_env = getenv("TM_DIRECT_STATIC");  // diagnostics: static tile assignment
    unsigned long long* ctr = (st_env && st_env[0] == '1') ? nullptr : next_tile_ctr();
    const bool range = !(off == 0 && n == g.P);
    cudaError_t e = tmx::launch_direct(shifted, g.k, n, g.strategy == TM_ASA16, g.sum, g.status, ctr, s,
                                       range ? g.range_ctas : 0);
    return e == cudaSuccess ? TM_OK : cuda_fail("launch_direct", e);
  }
  if (g.strategy == TM_AR) {
    if (!g.comm) return TM_E_NCCL;
    ncclResult_t r = g_nccl.AllReduce(bufs[0] + off, bufs[0] + off, (size_t)n, ncclFloat32,
                                      g.sum ? ncclSum : ncclAvg, g.comm, s);
    return r == ncclSuccess ? TM_OK : TM_E_NCCL;
  }
  ExchangeArgs a = make_args(bufs, off, n);
  return launch_staged(a, s);
}

// One BSP iteration: momentum-SGD step of every local rank, then the exchange
// of the weights (and of the velocities when exchange_momentum).
int do_bsp(float* const* w, float* const* v, const float* const* gr, int nbufs, float lr, float mu,
           int mom, cudaStream_t s) {
  if (!g.inited || !g.ready || g.strategy == TM_EASGD) return TM_E_STATE;
  if (g.sum) return TM_E_ARG;  // SUBGD sums updates, not weights: exchange deltas instead
  if (nbufs != g.nlocal || !w || !v || !gr) return TM_E_ARG;
  for (int i = 0; i < nbufs; ++i) {
    if (!w[i] || !v[i] || !gr[i]) return TM_E_ARG;
    if (!aligned16(w[i]) || !aligned16(v[i]) || !aligned16(gr[i])) return TM_E_ALIGN;
  }
  cudaSetDevice(g.device);
  const char* unf = getenv("TM_BSP_UNFUSED");  // diagnostics: time the unfused sequence
  const bool fuse = !(unf && unf[0] == '1');
  if (fuse && g.k > 1 && g.nlocal == g.k &&
      (g.strategy == TM_AR || effective_path() == TM_PATH_DIRECT)) {
    tmx::BspBufs bb{};
    for (int i = 0; i < nbufs; ++i) {
      bb.w[i] = w[i];
      bb.v[i] = v[i];
      bb.g[i] = gr[i];
    }
    bb.lr = lr;
    bb.mu = mu;
    cudaError_t e = tmx::launch_bsp_direct(bb, g.k, g.P, g.strategy == TM_ASA16, mom != 0, g.status,
                                           next_tile_ctr(), s);
    return e == cudaSuccess ? TM_OK : cuda_fail("launch_bsp_direct", e);
  }
  int rc = TM_OK;
  if (fuse && g.k > 1 && g.strategy != TM_AR) {
    // Staged path: the step is fused into the exchange's pre-cast (a2), which
    // reads w, v, g, writes v' and the wire staging of w' = w + v'; w' itself is
    // never written (the allgather overwrites every element of w).
    // With the momentum exchange (mom) the same launch also exchanges v': the
    // pre-cast writes v' to the wire as a second vector (not back to v), and
    // both vectors share the staging layout, the barriers and the launch.
    ExchangeArgs a = make_args(w, 0, g.P);
    for (int i = 0; i < nbufs; ++i) {
      a.v[i] = v[i];
      a.g[i] = gr[i];
    }
    a.lr = lr;
    a.mu = mu;
    a.sgd = 1;
    a.nvec = mom ? 2 : 1;
    return launch_staged(a, s);
  } else {
    for (int i = 0; i < nbufs; ++i) {
      cudaError_t e = tmx::launch_sgd(w[i], v[i], gr[i], g.P, lr, mu, s);
      if (e != cudaSuccess) return cuda_fail("launch_sgd", e);
    }
    if (g.k == 1) return TM_OK;  // reading Q10: the exchange is the identity
    rc = do_exchange(w, nbufs, 0, g.P, s);
  }
  if (rc != TM_OK || !mom) return rc;
  return do_exchange(v, nbufs, 0, g.P, s);
}

// ---------------------------------------------------------------------------
// Bootstrap known-answer self-check (one process per GPU).  The first staged
// exchange over the peer mappings is the first time this flavour's loads (for
// the TMA flavours: bulk copies of IPC-mapped peer memory over NVLink) run on
// this box, so before any caller data moves, every rank exchanges a probe whose
// average is exact by construction: x_r[i] = (m + r + 1) * 2^-8 with
// m = i mod 251, so the mean is (2m + k + 1) * 2^-9 (the sum k m + k(k+1)/2
// times 2^-8 in SUBGD sum mode) -- every value, every partial sum and the
// result have at most 11 significant bits, exact in binary16 and fp32 whatever
// the order.  Element-varying values catch misaddressed loads, rank-dependent
// ones a mixed-up peer.  Each rank compares its own result bit for bit, then
// the ranks vote through peer memory (each writes its verdict into every
// peer's pad tail with a copy through the IPC mapping and polls its own); if
// any rank failed, every rank falls back to the register flavour (plain 16-byte
// loads of peer memory), records it (tm_layout selfcheck = 2) and re-runs the
// probe on it.  A probe that times out is reported as TM_E_TIMEOUT.
// TM_SELFCHECK=0 skips it; TM_SELFCHECK_FAULT=r makes rank r report a mismatch
// (fault injection for the tests).
// ---------------------------------------------------------------------------
// CTAs per rank a cooperative launch of flavour fl can keep co-resident (all
// local ranks' grids at once).  TM_PROCS_PER_GPU=n: n processes share this GPU
// concurrently (CUDA MPS), so each may keep only 1/n of them (every rank's CTA c
// must be resident at once for the per-CTA flag barriers).
int flavour_cmax(int device, int strategy, int k, int nlocal, int fl) {
  const int share = std::max(1, getenv("TM_PROCS_PER_GPU") ? atoi(getenv("TM_PROCS_PER_GPU")) : 1);
  return tmx::exchange_max_ctas(device, wire16(strategy), k, fl) / nlocal / share;
}

uint32_t* pad_tail(int rank) {
  return reinterpret_cast<uint32_t*>(g.rank_base[rank] + g.off_flags +
                                     ((int64_t)tmx::kPhases * TM_MAX_RANKS + 1) * g.flag_c * 4);
}

int probe_once(float* probe, int64_t n, cudaStream_t st, bool* ok) {
  const float s8 = 1.0f / 256.0f;
  std::vector<float> h((size_t)n), back((size_t)n);
  for (int64_t i = 0; i < n; ++i) h[(size_t)i] = (float)((i % 251) + g.rank0 + 1) * s8;
  // Stream-ordered upload: a cudaMemcpy from pageable memory may return before
  // its DMA lands, and the probe runs on a non-blocking stream.
  cudaError_t e = cudaMemcpyAsync(probe, h.data(), (size_t)n * 4, cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return cuda_fail("probe upload", e);
  float* bufs[1] = {probe};
  ExchangeArgs a = make_args(bufs, 0, n);
  const uint64_t saved = g.timeout_ns;
  g.timeout_ns = std::min<uint64_t>(g.timeout_ns, 5ull * 1000 * 1000 * 1000);
  a.timeout_ns = g.timeout_ns;
  const int saved_ag = g.ag_mode;
  g.ag_mode = TM_AG_SM;  // the probe checks the kernel's own data path
  int rc = launch_staged(a, st);
  g.ag_mode = saved_ag;
  g.timeout_ns = saved;
  if (rc != TM_OK) return rc;
  e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return cuda_fail("probe sync", e);
  uint32_t bits = 0;
  e = cudaMemcpy(&bits, g.status, 4, cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return cuda_fail("probe status", e);
  e = cudaMemsetAsync(g.status, 0, 4, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return cuda_fail("probe status clear", e);
  if (bits & TM_BIT_TIMEOUT) return TM_E_TIMEOUT;
  e = cudaMemcpy(back.data(), probe, (size_t)n * 4, cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return cuda_fail("probe download", e);
  const int k = g.k;
  bool good = bits == 0;
  int64_t nbad = 0, first_bad = -1;
  for (int64_t i = 0; i < n; ++i) {
    const int64_t m = i % 251;
    const float want = g.sum ? (float)(k * m + k * (k + 1) / 2) * s8 : (float)(2 * m + k + 1) * (s8 * 0.5f);
    uint32_t wb, gb;
    memcpy(&wb, &want, 4);
    memcpy(&gb, &back[(size_t)i], 4);
    if (wb != gb) {
      if (first_bad < 0) first_bad = i;
      ++nbad;
    }
  }
  good = good && nbad == 0;
  if (!good && getenv("TM_DEBUG"))
    fprintf(stderr, "[tm] rank %d: self-check probe (flavour %d, n %lld, C %d): status bits %u, %lld of %lld "
                    "elements wrong, first at %lld (got %a)\n",
            g.rank0, g.staged_kernel, (long long)n, a.C, bits, (long long)nbad, (long long)n,
            (long long)first_bad, first_bad >= 0 ? (double)back[(size_t)first_bad] : 0.0);
  *ok = good;
  return TM_OK;
}

// Every rank's verdict for `round`, through the peers' pad tails.
int vote(uint32_t round, bool mine, bool* all) {
  const uint32_t v = (round << 8) | (mine ? 1u : 0u);
  for (int j = 0; j < g.k; ++j) {
    cudaError_t e = cudaMemcpy(pad_tail(j) + tmx::kTailVotes + g.rank0, &v, 4, cudaMemcpyDefault);
    if (e != cudaSuccess) return cuda_fail("vote", e);
  }
  uint32_t got[TM_MAX_RANKS];
  const auto t0 = std::chrono::steady_clock::now();
  for (;;) {
    cudaError_t e = cudaMemcpy(got, pad_tail(g.rank0) + tmx::kTailVotes, 4 * g.k, cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) return cuda_fail("vote poll", e);
    bool in = true, ok = true;
    for (int j = 0; j < g.k; ++j) {
      in = in && (got[j] >> 8) == round;
      ok = ok && (got[j] & 1u);
    }
    if (in) {
      *all = ok;
      return TM_OK;
    }
    if (std::chrono::steady_clock::now() - t0 > std::chrono::nanoseconds(g.timeout_ns)) return TM_E_TIMEOUT;
    usleep(200);
  }
}

int self_check() {
  const char* off = getenv("TM_SELFCHECK");
  if ((off && off[0] == '0') || g.nprocs == 1 || (g.strategy != TM_ASA && g.strategy != TM_ASA16))
    return TM_OK;
  const int64_t n = std::min<int64_t>(g.P, (int64_t)g.k * 8192);
  float* probe = nullptr;
  cudaError_t e = cudaMalloc(&probe, (size_t)n * 4);
  if (e != cudaSuccess) return cuda_fail("probe alloc", e);
  cudaStream_t st = nullptr;
  e = cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  if (e != cudaSuccess) {
    cudaFree(probe);
    return cuda_fail("probe stream", e);
  }
  const int fault = getenv("TM_SELFCHECK_FAULT") ? atoi(getenv("TM_SELFCHECK_FAULT")) : -1;
  int rc = TM_OK;
  for (uint32_t round = 1; round <= 2 && rc == TM_OK; ++round) {
    bool ok = false, all = false;
    rc = probe_once(probe, n, st, &ok);
    if (rc != TM_OK) break;
    if (round == 1 && fault == g.rank0) ok = false;  // fault injection
    rc = vote(round, ok, &all);
    if (rc != TM_OK) break;
    if (all) {
      g.selfcheck = round == 1 ? 1 : 2;
      break;
    }
    if (round == 2 || g.staged_kernel == tmx::kStagedReg) {
      rc = TM_E_MISMATCH;  // the plain flavour fails too: nothing left to fall back to
      break;
    }
    if (getenv("TM_DEBUG")) fprintf(stderr, "[tm] rank %d: self-check failed, register flavour\n", g.rank0);
    g.staged_kernel = tmx::kStagedReg;  // every rank takes the same decision (same votes)
    // C was sized for the failed flavour; the register kernel may keep fewer CTAs
    // co-resident (its cooperative launch would fail).  Every rank computes the
    // same C; the flag pad keeps its stride (flag_c).
    const int creg = flavour_cmax(g.device, g.strategy, g.k, g.nlocal, g.staged_kernel);
    if (creg < 1) {
      rc = TM_E_CUDA;
      break;
    }
    g.C = std::min(g.C, creg);
    g.Lc = round_up((g.L + g.C - 1) / g.C, tmx::kAlign);
  }
  cudaStreamDestroy(st);
  cudaFree(probe);
  return rc;
}

}  // namespace

extern "C" {

int tm_bsp_step(float* w, float* v, const float* grad, float lr, float mu,
                           int exchange_momentum, void* stream) {
  NvtxRange nvtx("tm_bsp_step");
  std::lock_guard<std::mutex> lk(g_mu);
  if (g.inited && g.nlocal != 1) return TM_E_STATE;
  float* ws[1] = {w};
  float* vs[1] = {v};
  const float* gs[1] = {grad};
  return do_bsp(ws, vs, gs, 1, lr, mu, exchange_momentum, static_cast<cudaStream_t>(stream));
}

int tm_bsp_step_group(float* const* w, float* const* v, const float* const* grad,
                                 int nbufs, float lr, float mu, int exchange_momentum,
                                 void* stream) {
  NvtxRange nvtx("tm_bsp_step_group");
  std::lock_guard<std::mutex> lk(g_mu);
  return do_bsp(w, v, grad, nbufs, lr, mu, exchange_momentum, static_cast<cudaStream_t>(stream));
}


int tm_exchange_init(int64_t nparams, const tm_world* world, int strategy) {
  std::lock_guard<std::mutex> lk(g_mu);
  if (g.inited) return TM_E_STATE;
  if (!world || nparams < 1) return TM_E_ARG;
  const bool op_sum = (strategy & TM_OP_SUM) != 0;
  strategy &= ~TM_OP_SUM;
  if (strategy < TM_AR || strategy > TM_EASGD) return TM_E_ARG;
  if (op_sum && strategy == TM_EASGD) return TM_E_ARG;
  const int k = world->size;
  if (k < 1 || k > TM_MAX_RANKS) return TM_E_ARG;
  if (world->nlocal != 1 && world->nlocal != k) return TM_E_ARG;
  if (world->rank < 0 || world->rank + world->nlocal > k) return TM_E_ARG;
  if (world->nlocal == k && world->rank != 0) return TM_E_ARG;
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess) return cuda_fail("cudaGetDeviceCount", e);
  if (world->device < 0 || world->device >= ndev) return TM_E_ARG;
  e = cudaSetDevice(world->device);
  if (e != cudaSuccess) return cuda_fail("cudaSetDevice", e);

  Ctx c;
  c.P = nparams;
  c.k = k;
  c.rank0 = world->rank;
  c.nlocal = world->nlocal;
  c.device = world->device;
  c.strategy = strategy;
  c.sum = op_sum;
  c.nprocs = k / world->nlocal;
  c.proc = world->rank / world->nlocal;
  c.L = round_up((nparams + k - 1) / k, tmx::kAlign);

  const int wb = wire_bytes(strategy);
  if (strategy == TM_ASA || strategy == TM_ASA16) {
    // Staged kernel flavour.  Single-process groups: the TMA-engine kernel
    // (measured fastest on one GPU).  Across processes: the warp-specialised
    // TMA-engine kernel, whose pre-cast (HBM) overlaps the reduce-scatter pull
    // (NVLink) sub-chunk by sub-chunk, both fed by bulk copies; on one GPU it
    // measures as the TMA kernel (0.982 vs 0.984 ms at AlexNet k = 8) and ahead
    // of the register warp-specialised kernel (1.248 ms).
    // TM_STAGED_KERNEL=reg|tma|ws|tmaws|oneshot|ll overrides (TM_STAGED_LDG=1 /
    // TM_STAGED_TMA=1 are accepted too).
    // Segments of at most TM_ONESHOT_MAX_L elements (default oneshot_max_l(k),
    // profiles/r02/latency/): the one-shot kernel (one barrier).  Up to
    // kRegMaxL: the register two-phase kernel, whose phases have no bulk-copy
    // round trips to drain (profiles/r01/latency_flavours.txt, r02/latency/).
    // Segments of at most TM_LL_MAX_L elements (default ll_max_l(k)): the LL
    // kernel, no barrier at all; up to TM_LL2_MAX_L (ll2_max_l(k)) the two-shot
    // LL2 kernel.
    const int64_t oneshot_max = env_i64("TM_ONESHOT_MAX_L", oneshot_max_l(k));
    const int64_t ll_max = env_i64("TM_LL_MAX_L", ll_max_l(k));
    const int64_t ll2_max = env_i64("TM_LL2_MAX_L", ll2_max_l(k));
    c.staged_kernel = c.L <= ll_max          ? tmx::kStagedLL
                      : c.L <= ll2_max       ? tmx::kStagedLL2
                      : c.L <= oneshot_max   ? tmx::kStagedOneShot
                      : c.L <= kRegMaxL      ? tmx::kStagedReg
                      : (c.nprocs == 1 ? tmx::kStagedTma : tmx::kStagedTmaWs);
    const char* sk = getenv("TM_STAGED_KERNEL");
    const char* ldg = getenv("TM_STAGED_LDG");
    const char* tma = getenv("TM_STAGED_TMA");
    if (ldg && ldg[0] == '1') c.staged_kernel = tmx::kStagedReg;
    if (tma && tma[0] == '1') c.staged_kernel = tmx::kStagedTma;
    if (sk && !strcmp(sk, "reg")) c.staged_kernel = tmx::kStagedReg;
    if (sk && !strcmp(sk, "tma")) c.staged_kernel = tmx::kStagedTma;
    if (sk && !strcmp(sk, "ws")) c.staged_kernel = tmx::kStagedWs;
    if (sk && !strcmp(sk, "tmaws")) c.staged_kernel = tmx::kStagedTmaWs;
    if (sk && !strcmp(sk, "oneshot")) c.staged_kernel = tmx::kStagedOneShot;
    if (sk && !strcmp(sk, "ll")) c.staged_kernel = tmx::kStagedLL;
    if (sk && !strcmp(sk, "ll2")) c.staged_kernel = tmx::kStagedLL2;
    const char* ag = getenv("TM_ALLGATHER");  // sm | ce | nccl
    const char* ag_table = getenv("TM_AG_TABLE");
    if (!ag && ag_table && c.nprocs > 1) ag = ag_table_mode(ag_table, k, c.L);
    if (ag && !strcmp(ag, "ce")) c.ag_mode = TM_AG_CE;
    c.want_nccl_ag = ag && !strcmp(ag, "nccl") && c.nprocs > 1;
    if (c.want_nccl_ag) c.ag_mode = TM_AG_NCCL;
    // co-resident CTAs per rank (TM_PROCS_PER_GPU: see flavour_cmax)
    int cmax = k >= 2 ? flavour_cmax(c.device, strategy, k, c.nlocal, c.staged_kernel) : 1;
    if (k >= 2 && cmax < 1) return TM_E_CUDA;
    const int64_t chunk = c.staged_kernel == tmx::kStagedOneShot ? oneshot_chunk() : tmx::kMinChunk;
    const bool ll = c.staged_kernel == tmx::kStagedLL || c.staged_kernel == tmx::kStagedLL2;
    const int64_t want = ll ? std::max<int64_t>(1, (nparams + tmx::kLLChunk - 1) / tmx::kLLChunk)
                            : std::max<int64_t>(1, (c.L + chunk - 1) / chunk);
    c.C = (int)std::min<int64_t>(std::max(cmax, 1), want);
    c.Lc = round_up((c.L + c.C - 1) / c.C, tmx::kAlign);
    c.flag_c = c.C;
    // The warp-specialised kernel overlaps the pre-cast with the pull only across
    // sub-chunks (>= kWsMinSub elements each); a chunk too short for two of them
    // would run both phases on half a CTA each with nothing to overlap, so the
    // TMA kernel (same shared memory, same C) takes it (k = 8 under MPS: 34.4 vs
    // 36.3 us at P = 1 Mi, 54.7 vs 58.0 us at 2 Mi; profiles/r02/latency/).
    if (c.staged_kernel == tmx::kStagedTmaWs && !(sk && *sk) && c.Lc < 2 * tmx::kWsMinSub)
      c.staged_kernel = tmx::kStagedTma;
    // Staging: nvec_alloc buffers of k*L wire elements (w, and v for the BSP step
    // with momentum exchange), twice over (call parity) for the one-shot kernel;
    // then nvec_alloc averaged segments of L; then the flag pad.
    c.nvec_alloc = 2;
    const bool twice = c.staged_kernel == tmx::kStagedOneShot || c.staged_kernel == tmx::kStagedLL ||
                       c.staged_kernel == tmx::kStagedLL2;
    const int nstage = twice ? 2 * c.nvec_alloc : c.nvec_alloc;
    c.stage_stride = round_up((int64_t)k * c.L * wb, 256);
    if (c.staged_kernel == tmx::kStagedLL) {
      // receive buffer per (parity, vector): k sources x LPS 16-byte lines, one
      // line per 4 elements (fp16 wire) or two (fp32 wire); the kernel derives
      // LPS = stage_stride / (16 k), which the staged flavours' own layout
      // (the register fallback of the self-check) also fits in
      const int64_t lps = round_up((nparams + 3) / 4, 16) * (wb == 2 ? 1 : 2);
      const int64_t unit = std::lcm<int64_t>(16 * (int64_t)k, 256);  // exact LPS, 256-byte aligned
      c.stage_stride = round_up(std::max<int64_t>(c.stage_stride, 16 * (int64_t)k * lps), unit);
    }
    if (c.staged_kernel == tmx::kStagedLL2) {
      // per (parity, vector): [reduce-scatter: k source slots][allgather: k owner
      // slots] of LPG lines (one segment's units); the kernel derives LPG =
      // stage_stride / (32 k)
      const int64_t lpg = round_up((c.L + 3) / 4, 16) * (wb == 2 ? 1 : 2);
      const int64_t unit = std::lcm<int64_t>(32 * (int64_t)k, 256);
      c.stage_stride = round_up(std::max<int64_t>(c.stage_stride, 32 * (int64_t)k * lpg), unit);
    }
    c.avg_stride = round_up(c.L * wb, 256);
    c.off_stage = 0;
    c.off_avg = c.off_stage + nstage * c.stage_stride;
    c.off_flags = c.off_avg + c.nvec_alloc * c.avg_stride;
    c.rank_stride = round_up(c.off_flags + ((int64_t)tmx::kPhases * TM_MAX_RANKS + 1) * c.flag_c * 4 +
                                 tmx::kPadTail * 4, 4096);
  } else if (strategy == TM_EASGD) {
    // Centre sharded by segment: rank s hosts c[s*L, min((s+1)*L, P)).
    c.off_center = 0;
    const int64_t nch = (c.L + tmx::kLockChunk - 1) / tmx::kLockChunk;
    c.off_locks = round_up(c.L * 4, 256);
    c.off_tickets = round_up(c.off_locks + nch * 4, 256);
    c.rank_stride = round_up(c.off_tickets + nch * 4, 4096);
  } else {
    c.rank_stride = 0;
  }
  // + status word (+0) and the ring of tile-claim counter pairs (+256)
  c.slab_bytes = c.rank_stride * c.nlocal + 256 + tmx::kCtrSlots * 16;
  e = cudaMalloc(reinterpret_cast<void**>(&c.slab), c.slab_bytes);
  if (e != cudaSuccess) return cuda_fail("cudaMalloc", e);
  // cudaMemset is asynchronous to the host (legacy stream): wait for it, so the
  // slab is zero before any kernel on a non-blocking stream, or any peer (after
  // the bootstrap), touches it.
  e = cudaMemset(c.slab, 0, c.slab_bytes);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    cudaFree(c.slab);
    return cuda_fail("cudaMemset", e);
  }
  c.status = reinterpret_cast<uint32_t*>(c.slab + c.rank_stride * c.nlocal);
  c.tile_ctrs = reinterpret_cast<unsigned long long*>(c.slab + c.rank_stride * c.nlocal + 256);
  c.range_ctas = std::max(0, getenv("TM_RANGE_CTAS") ? atoi(getenv("TM_RANGE_CTAS")) : 0);
  c.inited = true;
  c.ready = (c.nprocs == 1);
  g = c;
  fill_rank_bases_local();
  if ((g.strategy == TM_AR || g.want_nccl_ag) && g.nprocs > 1 && g.proc == 0) {
    if (!g_nccl.load()) {
      release();
      return TM_E_NCCL;
    }
    if (g_nccl.GetUniqueId(&g.nccl_id) != ncclSuccess) {
      release();
      return TM_E_NCCL;
    }
    g.have_nccl_id = true;
  }
  return TM_OK;
}

int tm_bootstrap_export(void* blob, size_t* len) {
  std::lock_guard<std::mutex> lk(g_mu);
  if (!g.inited) return TM_E_STATE;
  if (!blob || !len) return TM_E_ARG;
  Blob b;
  memset(&b, 0, sizeof(b));
  b.magic = kMagic;
  b.version = kVersion;
  b.rank0 = g.rank0;
  b.nlocal = g.nlocal;
  b.size = g.k;
  b.strategy = g.strategy | (g.sum ? TM_OP_SUM : 0);
  b.C = g.C;
  b.pid = (int32_t)getpid();
  b.P = g.P;
  b.L = g.L;
  b.Lc = g.Lc;
  b.rank_stride = g.rank_stride;
  b.off_stage = g.off_stage;
  b.off_avg = g.off_avg;
  b.off_flags = g.off_flags;
  b.off_center = g.off_center;
  b.device_ordinal = g.device;
  b.ag_nccl = g.want_nccl_ag ? 1 : 0;
  b.staged_kernel = g.staged_kernel;
  b.ag_mode = g.ag_mode;
  cudaSetDevice(g.device);
  cudaError_t e = cudaIpcGetMemHandle(&b.handle, g.slab);
  if (e != cudaSuccess) return cuda_fail("cudaIpcGetMemHandle", e);
  if (g.have_nccl_id) {
    b.has_nccl = 1;
    b.nccl_id = g.nccl_id;
  }
  memset(blob, 0, TM_BLOB_BYTES);
  memcpy(blob, &b, sizeof(b));
  *len = TM_BLOB_BYTES;
  return TM_OK;
}

int tm_bootstrap_import(const void* blobs, size_t len_each) {
  std::lock_guard<std::mutex> lk(g_mu);
  if (!g.inited) return TM_E_STATE;
  if (g.ready) return TM_OK;
  if (!blobs || len_each < sizeof(Blob)) return TM_E_ARG;
  cudaSetDevice(g.device);
  const char* p = static_cast<const char*>(blobs);
  const Blob* nccl_blob = nullptr;
  for (int q = 0; q < g.nprocs; ++q) {
    Blob b;
    memcpy(&b, p + (size_t)q * len_each, sizeof(b));
    if (b.magic != kMagic || b.version != kVersion) return TM_E_ARG;
    if (b.P != g.P || b.size != g.k || b.strategy != (g.strategy | (g.sum ? TM_OP_SUM : 0)) ||
        b.C != g.C || b.L != g.L ||
        b.Lc != g.Lc || b.nlocal != g.nlocal || b.rank_stride != g.rank_stride ||
        b.ag_nccl != (g.want_nccl_ag ? 1 : 0) || b.staged_kernel != g.staged_kernel ||
        b.ag_mode != g.ag_mode || b.rank0 != q * g.nlocal)
      return TM_E_MISMATCH;
    if (b.has_nccl) nccl_blob = reinterpret_cast<const Blob*>(p + (size_t)q * len_each);
    if (q == g.proc) continue;
    void* base = nullptr;
    cudaError_t e = cudaIpcOpenMemHandle(&base, b.handle, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) return cuda_fail("cudaIpcOpenMemHandle", e);
    g.peer_base[q] = static_cast<char*>(base);
    for (int i = 0; i < b.nlocal; ++i)
      g.rank_base[b.rank0 + i] = static_cast<char*>(base) + (int64_t)i * b.rank_stride;
  }
  if ((g.strategy == TM_AR || g.want_nccl_ag) && g.nprocs > 1) {
    if (!nccl_blob || !g_nccl.load()) return TM_E_NCCL;
    Blob nb;
    memcpy(&nb, nccl_blob, sizeof(nb));
    if (g_nccl.CommInitRank(&g.comm, g.nprocs, nb.nccl_id, g.proc) != ncclSuccess) return TM_E_NCCL;
  }
  g.ready = true;
  const int rc = self_check();
  if (rc != TM_OK) g.ready = false;
  return rc;
}

int tm_exchange(float* dev_buf, void* stream) {
  NvtxRange nvtx("tm_exchange");
  std::lock_guard<std::mutex> lk(g_mu);
  if (g.inited && g.nlocal != 1) return TM_E_STATE;
  float* bufs[1] = {dev_buf};
  return do_exchange(bufs, 1, 0, g.P, static_cast<cudaStream_t>(stream));
}

int tm_exchange_group(float* const* dev_bufs, int nbufs, void* stream) {
  NvtxRange nvtx("tm_exchange_group");
  std::lock_guard<std::mutex> lk(g_mu);
  return do_exchange(dev_bufs, nbufs, 0, g.P, static_cast<cudaStream_t>(stream));
}

int tm_exchange_range(float* dev_buf, int64_t offset, int64_t count, void* stream) {
  NvtxRange nvtx("tm_exchange_range");
  std::lock_guard<std::mutex> lk(g_mu);
  if (g.inited && g.nlocal != 1) return TM_E_STATE;
  float* bufs[1] = {dev_buf};
  return do_exchange(bufs, 1, offset, count, static_cast<cudaStream_t>(stream));
}

int tm_exchange_group_range(float* const* dev_bufs, int nbufs, int64_t offset, int64_t count,
                            void* stream) {
  NvtxRange nvtx("tm_exchange_group_range");
  std::lock_guard<std::mutex> lk(g_mu);
  return do_exchange(dev_bufs, nbufs, offset, count, static_cast<cudaStream_t>(stream));
}

int tm_easgd_update(float* worker_buf, float* center_buf, float alpha, void* stream) {
  int64_t n;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    if (!g.inited) return TM_E_STATE;
    n = g.P;
  }
  return tm_easgd_update_ex(worker_buf, center_buf, n, alpha, 0, stream);
}

int tm_easgd_update_ex(float* worker_buf, float* center_buf, int64_t n, float alpha,
                       int concurrent, void* stream) {
  NvtxRange nvtx("tm_easgd_update_ex");
  if (!worker_buf || !center_buf || n < 0) return TM_E_ARG;
  if (n == 0) return TM_OK;
  if ((reinterpret_cast<uintptr_t>(worker_buf) | reinterpret_cast<uintptr_t>(center_buf)) & 3)
    return TM_E_ALIGN;
  if (concurrent < 0 || concurrent > 2) return TM_E_ARG;
  cudaError_t e = tmx::launch_easgd(worker_buf, center_buf, n, alpha, concurrent,
                                   static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? TM_OK : cuda_fail("easgd", e);
}

int tm_easgd_round(float* const* workers, int nworkers, const int32_t* order, int norder,
                   float* center_buf, int64_t n, float alpha, void* stream) {
  NvtxRange nvtx("tm_easgd_round");
  if (!workers || !order || !center_buf || n < 0 || nworkers < 1 || nworkers > 16 ||
      norder < 0 || norder > 64)
    return TM_E_ARG;
  for (int i = 0; i < nworkers; ++i) {
    if (!workers[i]) return TM_E_ARG;
    if (reinterpret_cast<uintptr_t>(workers[i]) & 3) return TM_E_ALIGN;
  }
  for (int t = 0; t < norder; ++t)
    if (order[t] < 0 || order[t] >= nworkers) return TM_E_ARG;
  if (n == 0 || norder == 0) return TM_OK;
  cudaError_t e = tmx::launch_easgd_round(workers, nworkers, order, norder, center_buf, n, alpha,
                                         static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? TM_OK : cuda_fail("easgd_round", e);
}

int tm_easgd_center(int owner_rank, float** center) {
  std::lock_guard<std::mutex> lk(g_mu);
  if (!g.inited || !g.ready || g.strategy != TM_EASGD) return TM_E_STATE;
  if (!center || owner_rank < 0 || owner_rank >= g.k) return TM_E_ARG;
  *center = reinterpret_cast<float*>(g.rank_base[owner_rank] + g.off_center);
  return TM_OK;
}

int tm_easgd_update_sharded(float* worker_buf, float alpha, int concurrent, void* stream) {
  NvtxRange nvtx("tm_easgd_update_sharded");
  tmx::ShardArgs sa{};
  {
    std::lock_guard<std::mutex> lk(g_mu);
    if (!g.inited || !g.ready || g.strategy != TM_EASGD) return TM_E_STATE;
    if (!worker_buf) return TM_E_ARG;
    if (!aligned16(worker_buf)) return TM_E_ALIGN;
    for (int s = 0; s < g.k; ++s)
      sa.shard[s] = reinterpret_cast<float*>(g.rank_base[s] + g.off_center);
    sa.k = g.k;
    sa.L = g.L;
    sa.P = g.P;
    // a remote shard needs system-scope atomics when peers live in other processes
    sa.sys = g.nprocs > 1;
    cudaSetDevice(g.device);
  }
  if (concurrent < 0 || concurrent > 2) return TM_E_ARG;
  cudaError_t e = tmx::launch_easgd_sharded(worker_buf, sa, alpha, concurrent,
                                            static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? TM_OK : cuda_fail("easgd_sharded", e);
}

int tm_easgd_update_locked(float* worker_buf, int worker_id, float alpha, void* stream) {
  NvtxRange nvtx("tm_easgd_update_locked");
  tmx::ShardArgs sa{};
  {
    std::lock_guard<std::mutex> lk(g_mu);
    if (!g.inited || !g.ready || g.strategy != TM_EASGD) return TM_E_STATE;
    if (!worker_buf) return TM_E_ARG;
    if (!aligned16(worker_buf)) return TM_E_ALIGN;
    for (int s = 0; s < g.k; ++s) {
      sa.shard[s] = reinterpret_cast<float*>(g.rank_base[s] + g.off_center);
      sa.locks[s] = reinterpret_cast<uint32_t*>(g.rank_base[s] + g.off_locks);
      sa.tickets[s] = reinterpret_cast<uint32_t*>(g.rank_base[s] + g.off_tickets);
    }
    sa.order_log = g.order_log;
    sa.log_stride = g.order_log_stride;
    sa.worker_id = worker_id;
    sa.k = g.k;
    sa.L = g.L;
    sa.P = g.P;
    sa.sys = g.nprocs > 1;
    sa.status = g.status;
    sa.timeout_ns = g.timeout_ns;
    cudaSetDevice(g.device);
  }
  cudaError_t e = tmx::launch_easgd_locked(worker_buf, sa, alpha, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? TM_OK : cuda_fail("easgd_locked", e);
}

int tm_easgd_set_order_log(int32_t* dev_log, int max_updates_per_chunk) {
  std::lock_guard<std::mutex> lk(g_mu);
  if (!g.inited || g.strategy != TM_EASGD) return TM_E_STATE;
  if (dev_log && max_updates_per_chunk < 1) return TM_E_ARG;
  g.order_log = dev_log;
  g.order_log_stride = dev_log ? max_updates_per_chunk : 0;
  if (!dev_log) return TM_OK;
  // restart the tickets so log positions start at 0
  cudaSetDevice(g.device);
  for (int i = 0; i < g.nlocal; ++i) {
    const int64_t nch = (g.L + tmx::kLockChunk - 1) / tmx::kLockChunk;
    cudaError_t e = cudaMemset(g.rank_base[g.rank0 + i] + g.off_tickets, 0, nch * 4);
    if (e != cudaSuccess) return cuda_fail("ticket reset", e);
  }
  const cudaError_t e = cudaDeviceSynchronize();  // the reset lands before any later launch
  return e == cudaSuccess ? TM_OK : cuda_fail("ticket reset sync", e);
}

int tm_exchange_status(void* stream, uint32_t* bits) {
  std::lock_guard<std::mutex> lk(g_mu);
  if (!g.inited) return TM_E_STATE;
  cudaSetDevice(g.device);
  cudaError_t e = cudaStreamSynchronize(static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail("cudaStreamSynchronize", e);
  uint32_t h = 0;
  e = cudaMemcpy(&h, g.status, 4, cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return cuda_fail("status copy", e);
  // cleared on the caller's stream and waited for: a cudaMemset (legacy stream)
  // could land after the next exchange on a non-blocking stream set a bit
  e = cudaMemsetAsync(g.status, 0, 4, static_cast<cudaStream_t>(stream));
  if (e == cudaSuccess) e = cudaStreamSynchronize(static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail("status clear", e);
  if (bits) *bits = h;
  if (h & TM_BIT_TIMEOUT) return TM_E_TIMEOUT;
  if (h & TM_BIT_OVERFLOW16) return TM_E_OVERFLOW16;
  if (h & TM_BIT_NONFINITE) return TM_E_NONFINITE;
  return TM_OK;
}

int tm_layout(tm_layout_info* out) {
  std::lock_guard<std::mutex> lk(g_mu);
  if (!g.inited) return TM_E_STATE;
  if (!out) return TM_E_ARG;
  memset(out, 0, sizeof(*out));
  out->nparams = g.P;
  out->seg_len = g.L;
  out->chunk_len = g.Lc;
  out->k = g.k;
  out->rank = g.rank0;
  out->nlocal = g.nlocal;
  out->strategy = g.strategy | (g.sum ? TM_OP_SUM : 0);
  out->ctas_per_rank = g.C;
  out->threads = tmx::kThreads;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, g.device);
  out->sm_count = sms;
  out->wire_bytes = wire_bytes(g.strategy);
  out->lib_bytes = g.slab_bytes;
  out->epoch = g.epoch;
  out->path = effective_path();
  out->staged_kernel = g.staged_kernel;
  out->allgather = g.ag_mode;
  out->selfcheck = g.selfcheck;
  return TM_OK;
}

int tm_set_allgather(int mode) {
  std::lock_guard<std::mutex> lk(g_mu);
  if (!g.inited) return TM_E_STATE;
  if (mode < TM_AG_SM || mode > TM_AG_NCCL) return TM_E_ARG;
  if (mode == TM_AG_NCCL && !g.comm) return TM_E_NCCL;
  g.ag_mode = mode;
  return TM_OK;
}

int tm_set_path(int path) {
  std::lock_guard<std::mutex> lk(g_mu);
  if (!g.inited) return TM_E_STATE;
  if (path < TM_PATH_AUTO || path > TM_PATH_DIRECT) return TM_E_ARG;
  if (path == TM_PATH_DIRECT && g.nlocal != g.k) return TM_E_ARG;
  g.path = path;
  return TM_OK;
}

int tm_set_phase_log(uint64_t* dev_buf, int64_t capacity) {
  std::lock_guard<std::mutex> lk(g_mu);
  if (!g.inited) return TM_E_STATE;
  if (dev_buf && capacity < 1) return TM_E_ARG;
  g.stamps = dev_buf;
  g.stamps_cap = dev_buf ? capacity : 0;
  return TM_OK;
}

int tm_set_range_ctas(int ctas) {
  std::lock_guard<std::mutex> lk(g_mu);
  if (!g.inited) return TM_E_STATE;
  if (ctas < 0) return TM_E_ARG;
  g.range_ctas = ctas;
  return TM_OK;
}

int tm_set_timeout_ns(uint64_t ns) {
  std::lock_guard<std::mutex> lk(g_mu);
  g.timeout_ns = ns ? ns : kDefaultTimeoutNs;
  return TM_OK;
}

int tm_exchange_finalize(void) {
  std::lock_guard<std::mutex> lk(g_mu);
  if (g.inited) {
    cudaSetDevice(g.device);
    cudaDeviceSynchronize();
  }
  release();
  return TM_OK;
}

const char* tm_strerror(int status) {
  switch (status) {
    case TM_OK: return "ok";
    case TM_E_ARG: return "invalid argument";
    case TM_E_ALIGN: return "device buffer not 16-byte aligned";
    case TM_E_STATE: return "call out of order (init/bootstrap state)";
    case TM_E_CUDA: return "CUDA error";
    case TM_E_NCCL: return "NCCL unavailable or failed";
    case TM_E_MISMATCH: return "ranks disagree on nparams/strategy/layout";
    case TM_E_TIMEOUT: return "peer did not arrive before the timeout";
    case TM_E_NONFINITE: return "non-finite input element";
    case TM_E_OVERFLOW16: return "input overflows binary16 (|x| >= 65520)";
    case TM_E_IO: return "batch file missing, truncated or of the wrong shape";
    default: return "unknown status";
  }
}

int tm_cast_rn16(const float* in, uint16_t* out16, int64_t n, void* stream) {
  if (!in || !out16 || n < 0) return TM_E_ARG;
  if (n == 0) return TM_OK;
  cudaError_t e = tmx::launch_cast_rn16(in, out16, n, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? TM_OK : cuda_fail("cast_rn16", e);
}

}  // extern "C"
