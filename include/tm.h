/*
 * tm.h -- C ABI of libtm.so: the B200-native BSP parameter exchange of Theano-MPI
 * (Ma, Mao, Taylor; arXiv 1605.08325).  Plain C types only (no torch, no CUDA
 * headers): device buffers are `float*`, streams are `void*` holding a
 * cudaStream_t (e.g. torch.cuda.current_stream().cuda_stream; NULL = legacy
 * default stream).
 *
 * What is computed (PAPER.md = /root/reference/PAPER.md, line numbers):
 *   L66-70, L195-212  BSP data parallelism: after each SGD step the k workers'
 *                     parameters are "exchanged between worker processes in a
 *                     collective way"; L377-384 (AWAGD) averages them (1/k).
 *   L227-228          "Synchronous parameter exchange is an array reduction problem".
 *   L233-237          AR    : MPI Allreduce().
 *   L237-246, L252-256 ASA  : Alltoall of k sub-arrays, GPU summation on the owner,
 *                     Allgather of the sums.
 *   L262-269          ASA16 : ASA with the transfers in half precision, the
 *                     summation in full precision.
 *   L143-148, L573-588 EASGD : elastic averaging of a worker and a centre
 *                     (update equations: SPEC.md L475).
 *
 * Result of one tm_exchange, per element i, identical on every rank (DESIGN.md
 * readings Q1-Q10):
 *   ASA, AR : s = x_0[i]; s = fl(s + x_j[i]) for j = 1..k-1 (ascending rank);
 *             out = fl(s / k).   (AR through NCCL: order not fixed, see below.)
 *   ASA16   : h_j = rn16(x_j[i]) for every j (own included); s = widen(h_0);
 *             s = fl(s + widen(h_j)) ascending; a = fl(s / k);
 *             out = widen(rn16(a)) on every rank (owner included).
 *   rn16 = IEEE binary16 round-to-nearest-even, gradual subnormals, |x| >= 65520
 *   -> +-inf; widen exact; fl = one IEEE fp32 operation, no FMA, no FTZ.
 *   k = 1: identity for every strategy (nothing launched).
 *
 * Layout: rank r owns segment r = elements
 * [r*L, min((r+1)*L, P)), L = roundup(ceil(P/k), 256); padding is +0 and never
 * written to the caller's buffer.  The library owns all staging (k*L wire
 * elements per rank), the owner's averaged segment (L wire elements), the flag
 * pad and the status word, allocated with cudaMalloc at init (required for CUDA
 * IPC export) and freed at finalize.
 *
 * Process model: one exchanger per process.  A process hosts `nlocal`
 * consecutive ranks [rank, rank + nlocal) on ONE device:
 *   nlocal == 1     -- one process per GPU (torchrun); peers are reached through
 *                      CUDA IPC mappings over NVLink/NVSwitch.  Needs the
 *                      bootstrap (export -> all-gather of blobs -> import).
 *   nlocal == size  -- a single-process group: all k ranks' buffers live on one
 *                      device ("k simulated workers").  No bootstrap.  By default
 *                      the one-pass direct path runs (tm_path below); the
 *                      staged kernels run too (TM_PATH_STAGED), with local
 *                      pointers in the peer table.
 * Thread safety: one host thread per process calls tm_*.
 *
 * Environment (read at tm_exchange_init unless noted; every rank of a group must
 * use the same values):
 *   TM_STAGED_KERNEL=reg|tma|ws|tmaws|oneshot|ll|ll2  staged kernel flavour (default:
 *                      ll for segments L <= TM_LL_MAX_L elements (default
 *                      512 Ki at k = 2, 64 Ki at k <= 4, 8 Ki above), ll2 for
 *                      L <= TM_LL2_MAX_L (1 Mi, 256 Ki, 64 Ki), then
 *                      oneshot for L <= TM_ONESHOT_MAX_L elements
 *                      (default 1 Mi at k = 2, 32 Ki at k <= 4, 16 Ki above),
 *                      reg for L <= 32 Ki, else tma in a single-process group
 *                      and tmaws across processes).
 *   TM_ALLGATHER=sm|ce|nccl            allgather mode (tm_set_allgather); nccl
 *                      also creates the NCCL communicator at bootstrap.
 *   TM_AG_TABLE=path                   without TM_ALLGATHER: the mode by (k, L)
 *                      from a table measured on the multi-GPU box, one rule
 *                      "k L_max mode" per line, first match wins (default sm).
 *   TM_PROCS_PER_GPU=n                 n processes share this GPU concurrently
 *                      (CUDA MPS): each keeps 1/n of the co-resident CTAs.
 *   TM_NCCL_LIB=path                   libnccl.so.2 to dlopen (the binding sets
 *                      torch's); TM_DEBUG=1 prints CUDA errors to stderr.
 *   Diagnostics (read at first use): TM_DIRECT_LDG=1 register kernels instead of
 *   the TMA ones on the direct / BSP / EASGD-round paths; TM_DIRECT_TMA=1 the
 *   TMA direct kernel also for small exchanges (k * P <= 8 Mi elements, which
 *   use the register kernel by default: latency-bound); TM_DIRECT_STATIC=1
 *   static tile assignment; TM_TMA_CFG=n direct-kernel tile/ring variant;
 *   TM_BSP_UNFUSED=1 SGD pass + exchange instead of the fused kernels.
 *
 * Collective contract: every rank calls tm_exchange the same
 * number of times, in the same order.  Each call carries an epoch (kept on the
 * device, per CTA, so exchanges can be captured in CUDA graphs); cross-rank
 * synchronisation is by per-CTA epoch flags in peer memory (st.release /
 * ld.acquire at system scope across processes, GPU scope within one).  A rank
 * that never arrives makes its peers' spins time out: they set TM_E_TIMEOUT in
 * the sticky status and exit (no hang); the exchanger must then be re-created.
 *
 * Errors: argument/state/launch errors are returned synchronously.  Numeric
 * conditions never abort the collective; they set sticky status bits read by
 * tm_exchange_status: non-finite inputs (TM_E_NONFINITE), fp16 overflow of an
 * input, |x| >= 65520 (TM_E_OVERFLOW16, ASA16; the value becomes +-inf as IEEE
 * prescribes), barrier timeout (TM_E_TIMEOUT).
 */
#ifndef TM_H_
#define TM_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TM_MAX_RANKS 8      /* one NVSwitch box */
#define TM_BLOB_BYTES 512   /* size of one bootstrap blob */

/* OR into the strategy of tm_exchange_init: SUBGD, "summing up the parameter
 * updates from all GPUs before performing gradient descent" (PAPER L384-389,
 * the mode of the paper's runs, L458-460): the exchange returns the rank-order
 * fp32 sum instead of the average (no 1/k); ASA16 rounds the sum to binary16
 * (TM_E_OVERFLOW16 if it leaves the range).  Not valid with TM_EASGD. */
#define TM_OP_SUM 0x100

typedef enum {
  TM_AR = 0,     /* plain allreduce                     */
  TM_ASA = 1,    /* Alltoall-sum-Allgather, fp32 wire (L237-246)          */
  TM_ASA16 = 2,  /* ASA with fp16 wire, fp32 summation (L262-269)         */
  TM_EASGD = 3   /* EASGD context: library-owned centre buffer (L573-588) */
} tm_strategy;

typedef enum {
  TM_OK = 0,
  TM_E_ARG = 1,        /* bad argument (null, size, rank, strategy)               */
  TM_E_ALIGN = 2,      /* a device buffer is not 16-byte aligned                   */
  TM_E_STATE = 3,      /* call out of order (not initialised / not bootstrapped)  */
  TM_E_CUDA = 4,       /* a CUDA runtime call or launch failed                     */
  TM_E_NCCL = 5,       /* NCCL missing or failed (AR across processes)            */
  TM_E_MISMATCH = 6,   /* ranks disagree on nparams / strategy / layout           */
  TM_E_TIMEOUT = 7,    /* a peer did not arrive within the timeout (sticky)       */
  TM_E_NONFINITE = 8,  /* a non-finite input element was seen (sticky)             */
  TM_E_OVERFLOW16 = 9, /* an input rounded to +-inf in binary16 (sticky, ASA16)   */
  TM_E_IO = 10         /* loader: batch file missing, truncated or of wrong shape  */
} tm_status;

/* Sticky status bits (tm_exchange_status's `bits`). */
#define TM_BIT_NONFINITE 0x1u
#define TM_BIT_OVERFLOW16 0x2u
#define TM_BIT_TIMEOUT 0x4u
#define TM_BIT_LOG_OVERFLOW 0x8u /* test hook: a chunk saw more locked updates than the order log holds */

typedef struct {
  int32_t rank;    /* first global rank hosted by this process                */
  int32_t size;    /* k, number of ranks (workers), 1..TM_MAX_RANKS           */
  int32_t device;  /* CUDA device ordinal used by this process               */
  int32_t nlocal;  /* ranks hosted by this process: 1 or size (see above)     */
} tm_world;

typedef struct {
  int64_t nparams;       /* P                                                 */
  int64_t seg_len;       /* L = roundup(ceil(P/k), 256)                      */
  int64_t chunk_len;     /* per-CTA slice of a segment (multiple of 256)      */
  int32_t k, rank, nlocal, strategy;
  int32_t ctas_per_rank; /* C: CTAs per rank in the exchange kernel           */
  int32_t threads;       /* threads per CTA                                   */
  int32_t sm_count;
  int32_t wire_bytes;    /* 4 (AR, ASA) or 2 (ASA16)                          */
  int64_t lib_bytes;     /* device bytes the library owns in this process     */
  uint32_t epoch;        /* number of staged exchanges issued so far          */
  int32_t path;          /* effective tm_path of the next exchange            */
  int32_t staged_kernel; /* staged flavour: 0 register, 1 TMA engine, 2 warp-specialised,
                            3 warp-specialised on the TMA engine, 4 one-shot,
                            5 low-latency (LL: epoch inside every line, no barrier),
                            6 two-shot LL (push to the owner, owner pushes the average) */
  int32_t allgather;     /* tm_allgather mode of the staged path                */
  int32_t selfcheck;     /* bootstrap known-answer check: 0 not run, 1 passed,
                            2 the chosen flavour failed and every rank fell back
                            to the register flavour (staged_kernel = 0)        */
} tm_layout_info;

/* How an ASA / ASA16 exchange moves data (results are bitwise identical):
 *   TM_PATH_STAGED  pre-cast into library-owned staging, flag barrier,
 *                   reduce-scatter PULL from every rank's staging (NVLink P2P
 *                   loads across GPUs), flag barrier, allgather PULL.  The wire
 *                   carries fp16 for ASA16.  Required when ranks live in
 *                   different processes (nlocal == 1).
 *   TM_PATH_DIRECT  single-process groups only (nlocal == size): one pass in
 *                   which the owner of each element pulls the k fp32
 *                   contributions straight from the k caller buffers, applies
 *                   the same arithmetic (rn16 of each contribution for ASA16,
 *                   ascending-rank sum, /k, rn16) in registers and pushes the
 *                   result to all k buffers: no staging, no flags.
 *   TM_PATH_AUTO    DIRECT when nlocal == size, else STAGED (default). */
typedef enum { TM_PATH_AUTO = 0, TM_PATH_STAGED = 1, TM_PATH_DIRECT = 2 } tm_path;

/* How the staged path's allgather ("Allgather
 * ... do[es] not involve any arithmetic") moves the averaged segments; results
 * are bitwise identical in every mode:
 *   TM_AG_SM    (default) the exchange kernel's CTAs pull every rank's averaged
 *               segment over NVLink and widen it into the caller's buffer, fused.
 *   TM_AG_CE    the kernel stops after the reduced barrier; the COPY ENGINES
 *               gather the k averaged segments (cudaMemcpyAsync from the peer
 *               mappings into the library's staging, k copies per rank), then a
 *               widen kernel writes the caller's buffer (ASA: the copies land in
 *               the caller's buffer directly).  Frees the SMs during the gather.
 *   TM_AG_NCCL  as TM_AG_CE with ncclAllGather of the segments (the north
 *               star's "falling back to NCCL allgather over NVLink only where it
 *               measures faster").  Needs an NCCL communicator: processes that
 *               set TM_ALLGATHER=nccl in the environment before tm_exchange_init
 *               get one at bootstrap (one process per GPU, nlocal == 1). */
typedef enum { TM_AG_SM = 0, TM_AG_CE = 1, TM_AG_NCCL = 2 } tm_allgather;

/* Create the process-global exchanger.  nparams >= 1; world as above; strategy
 * a tm_strategy.  Allocates the library-owned buffers on world->device.  For
 * nlocal == size the exchanger is ready on return; otherwise the bootstrap
 * below must follow.  The buffers are zeroed before the call returns (the
 * first exchange may run on any stream, and peers write into them after the
 * bootstrap).  Returns TM_OK, TM_E_ARG, TM_E_STATE (already initialised) or
 * TM_E_CUDA. */
int tm_exchange_init(int64_t nparams, const tm_world* world, int strategy);

/* Write this process's bootstrap blob (CUDA IPC handle of its slab, layout, and
 * on the process hosting rank 0 an NCCL unique id for AR) into `blob`, which
 * must hold TM_BLOB_BYTES; *len receives TM_BLOB_BYTES. */
int tm_bootstrap_export(void* blob, size_t* len);

/* `blobs` holds size/nlocal blobs of `len_each` bytes, in process order
 * (process p hosts ranks [p*nlocal, (p+1)*nlocal)).  Opens the peers' IPC
 * mappings, checks that every process agrees on nparams, strategy, layout,
 * staged flavour and allgather mode (else TM_E_MISMATCH), and for AR
 * initialises the NCCL communicator (collective: every process must call it).
 * ASA / ASA16 then run a known-answer self-check of the staged flavour over the
 * peer mappings: a probe exchange whose average is exact by construction,
 * checked bit for bit on every rank, with a vote through peer memory; if any
 * rank fails, all ranks fall back to the register flavour (tm_layout
 * selfcheck = 2).  TM_E_TIMEOUT if the probe or the vote times out,
 * TM_E_MISMATCH if the register flavour fails too.  TM_SELFCHECK=0 skips it. */
int tm_bootstrap_import(const void* blobs, size_t len_each);

/* North-star call: average dev_buf (fp32[nparams], this rank's device, 16-byte
 * aligned, caller-owned) across the k ranks, IN PLACE, on `stream`.
 * Asynchronous: returns after enqueueing.  Requires nlocal == 1. */
int tm_exchange(float* dev_buf, void* stream);

/* Same for a process hosting nlocal ranks: dev_bufs is a HOST array of nbufs ==
 * nlocal device pointers (rank order), each fp32[nparams], 16-byte aligned,
 * pairwise disjoint. */
int tm_exchange_group(float* const* dev_bufs, int nbufs, void* stream);

/* Exchange only elements [offset, offset + count) of the buffer(s): a bucket,
 * e.g. one layer's parameters, so that buckets can be exchanged while backward
 * is still producing the next ones -- the overlap the paper leaves as future
 * work.  Same result as tm_exchange on those
 * elements (the method is elementwise); the range is partitioned into k
 * segments of its own.  offset must be a multiple of 4 (16-byte alignment),
 * 0 <= offset, offset + count <= nparams.  Ranges of one exchanger are
 * serialised by stream order: issue them on one stream, or order streams with
 * events; every rank issues the same ranges in the same order. */
int tm_exchange_range(float* dev_buf, int64_t offset, int64_t count, void* stream);
int tm_exchange_group_range(float* const* dev_bufs, int nbufs, int64_t offset, int64_t count,
                            void* stream);

/* One BSP iteration's update + combine (PAPER L195-212,
 * L373-384): every rank takes its momentum-SGD step (one IEEE
 * rounding per operation, no FMA):
 *     v = fl(fl(mu*v) - fl(lr*grad));   w = fl(w + v)
 * and then the weights are exchanged (averaged) with the exchanger's strategy;
 * exchange_momentum != 0 also averages the velocities (PAPER L160-164,
 * L373-376), else each rank keeps its own.  w, v, grad: fp32[nparams], 16-byte
 * aligned; w and v are updated in place.  In a single-process group on the
 * direct path the step and the exchange are ONE fused pass over memory; on the
 * staged path (across processes / GPUs) the step is fused into the exchange
 * kernel's pre-cast: it reads w, v, grad, writes v' and the wire staging of
 * w' = w + v' (w' itself is only written by the allgather).  On a timeout
 * (TM_E_TIMEOUT) w is left unspecified.
 * Not valid with TM_OP_SUM (exchange the updates with tm_exchange instead). */
int tm_bsp_step(float* w, float* v, const float* grad, float lr, float mu, int exchange_momentum,
                void* stream);
int tm_bsp_step_group(float* const* w, float* const* v, const float* const* grad, int nbufs,
                      float lr, float mu, int exchange_momentum, void* stream);

/* North-star call: one elastic update of nparams elements:
 *   d = fl(x - c); e = fl(alpha*d); x = fl(x - e); c = fl(c + e)   (no FMA)
 * worker_buf: this rank's fp32 buffer; center_buf: any fp32 buffer addressable
 * from this device (local, or from tm_easgd_center).  The caller guarantees
 * exclusive access to the centre for the duration (serialised server order,
 * reading Q15).  Works in any initialised context; n = init nparams. */
int tm_easgd_update(float* worker_buf, float* center_buf, float alpha, void* stream);

/* Extended form: explicit length n, and a concurrent mode so several workers
 * may update one centre at once (no lost updates; order not fixed):
 *   concurrent = 0  exclusive (the caller serialises the workers);
 *   concurrent = 1  centre += e by the hardware float atomic
 *                   (red.global.add(.v4).f32, system scope): it flushes
 *                   fp32-subnormal operands and results of the centre's add to
 *                   signed zero, unlike the exclusive update;
 *   concurrent = 2  centre += e by a compare-and-swap loop around one IEEE
 *                   fp32 add (gradual underflow, reading Q6): every update is
 *                   exactly fl(c + e) of the value it replaced.  A centre on
 *                   this GPU takes one 128-bit CAS per 4 elements (16-byte
 *                   aligned buffers; 1.31 vs 1.15 ms for concurrent = 1 at
 *                   config 4); peer memory one 32-bit CAS per element (3.42
 *                   ms).  TM_EASGD_CAS128=0 forces the 32-bit CAS.
 * TM_E_ARG for another value.  Does not need tm_exchange_init. */
int tm_easgd_update_ex(float* worker_buf, float* center_buf, int64_t n, float alpha,
                       int concurrent, void* stream);

/* A whole server round on one device, in ARRIVAL order ("without
 * the Round-Robin scheme"): for t = 0..norder-1 apply the elastic update of
 * workers[order[t]] against the centre, in one fused pass over the elements.
 * Bitwise equal to norder serial tm_easgd_update calls.  workers: HOST array of
 * nworkers device pointers; order: HOST array of norder indices in
 * [0, nworkers); nworkers <= 16, norder <= 64.  Does not need init.
 * Rounds over disjoint buffers may run concurrently on different streams: each
 * launch claims its tiles from its own counter pair (a per-device ring of 64,
 * so at most 64 rounds may be in flight on a device at once). */
int tm_easgd_round(float* const* workers, int nworkers, const int32_t* order, int norder,
                   float* center_buf, int64_t n, float alpha, void* stream);

/* EASGD context (strategy TM_EASGD): the centre x~ is SHARDED by segment
 * (SURVEY 8(e)): rank s hosts c[s*L, min((s+1)*L, P)) (L = seg_len of
 * tm_layout), so k workers updating it spread the traffic over all k GPUs'
 * NVLink ports instead of funnelling it into one server GPU.
 * tm_easgd_center returns owner_rank's shard as a pointer usable on this device
 * (local, or IPC-mapped over NVLink); its length is max(0, min(L, P - owner*L)). */
int tm_easgd_center(int owner_rank, float** center);

/* One elastic update (as tm_easgd_update) of this worker's full fp32[nparams]
 * buffer against the sharded centre: element i meets the shard of rank i / L.
 * concurrent == 0: the caller serialises the workers (bitwise equal to the
 * oracle's arrival order); 1 / 2: centre += e by the float atomic / the
 * CAS-loop IEEE add of tm_easgd_update_ex (system scope across processes), no
 * lost updates, order not fixed; mode 2 takes the 128-bit CAS when every shard
 * is in this GPU's memory, the 32-bit CAS otherwise. */
int tm_easgd_update_sharded(float* worker_buf, float alpha, int concurrent, void* stream);

/* Per-worker ATOMIC exchange with the sharded centre (the server
 * never interleaves two half-completed exchanges; workers are
 * served in arrival order, no Round-Robin): the centre is updated in chunks of
 * 4096 elements, each under a spin lock (system-scope atomics across
 * processes), so several workers may call concurrently (any streams, any
 * processes) and every chunk ends up exactly as the serial EASGD sequence in
 * that chunk's arrival order.  worker_id is recorded in the order log (test
 * hook below).  A lock not obtained within the timeout sets TM_E_TIMEOUT. */
int tm_easgd_update_locked(float* worker_buf, int worker_id, float alpha, void* stream);

/* Test hook: record, for every (shard s, chunk q), the worker_ids of locked
 * updates in arrival order into dev_log[(s*nchunk + q)*max + t] (int32,
 * device memory owned by the caller, nchunk = ceil(seg_len/4096)); resets this
 * process's tickets.  Arrivals past `max` per chunk are not logged and set the
 * sticky status bit TM_BIT_LOG_OVERFLOW (tm_exchange_status).  NULL disables. */
int tm_easgd_set_order_log(int32_t* dev_log, int max_updates_per_chunk);

/* ----------------------------------------------------------------------------
 * Parallel loading (Algorithm 1).  A native
 * loader thread per training process reads batch files into pinned host memory
 * (hostdata_x), copies the RAW uint8 batch to the GPU, subtracts the mean image,
 * crops and mirrors there (gpudata_x), and at Alg. 1's synchronisation point
 * copies gpudata_x into the trainer's input_x and notifies the trainer.
 *
 * Batch file: "PXB1" | u32 n | u32 c | u32 h | u32 w (little endian)
 * | n*c*h*w uint8, NCHW.  Output input_x: fp32 [n][c][crop_h][crop_w],
 *   input_x[b][k][y][x] = fl(float(raw[b][k][oy+y][ox+xs]) - mean[k][oy+y][ox+xs]),
 *   xs = mirror ? crop_w-1-x : x.
 * Crop / mirror: TRAIN mode, per example b of the f-th file loaded since create
 * (f = 0, 1, ...): z = splitmix64(seed ^ splitmix64((f << 32) | b)),
 * oy = z % (h-crop_h+1), ox = (z >> 20) % (w-crop_w+1), mirror = (z >> 40) & 1;
 * VAL mode: centre crop ((h-crop_h)/2, (w-crop_w)/2), no mirror.
 * splitmix64(z): z += 0x9E3779B97F4A7C15; z = (z ^ z>>30) * 0xBF58476D1CE4E5B9;
 * z = (z ^ z>>27) * 0x94D049BB133111EB; return z ^ z>>31.
 *
 * Protocol (Alg. 1): send TRAIN or VAL, then the first FILE; every later FILE
 * (sent when training on the last input_x is done) releases the previously
 * loaded batch into input_x (tm_loader_wait returns once it is there) and
 * starts loading the new one.  A TRAIN / VAL / STOP message ends the inner loop
 * (the batch loaded last is not delivered) and is taken as the next mode
 * (reading Q20).  ------------------------------------------------------------ */
enum { TM_LOADER_TRAIN = 0, TM_LOADER_VAL = 1, TM_LOADER_STOP = 2, TM_LOADER_FILE = 3 };

typedef struct {
  int32_t n, c, h, w;      /* batch geometry: examples, channels, height, width   */
  int32_t crop_h, crop_w;  /* crop window (<= h, w)                                 */
  int32_t device;          /* CUDA device of input_x                                */
  uint64_t seed;           /* crop / mirror generator seed                          */
  const float* mean;       /* HOST fp32 mean image [c][h][w], copied at create      */
} tm_loader_config;

typedef struct tm_loader tm_loader;

/* input_x: trainer-owned device buffer of n*c*crop_h*crop_w floats. */
int tm_loader_create(const tm_loader_config* cfg, float* input_x, tm_loader** out);
/* kind: TM_LOADER_*; filename for TM_LOADER_FILE (copied). Non-blocking.
 * A FILE message releases the loaded batch into input_x (Alg. 1): the copy
 * is ordered after all work enqueued on `stream` (a cudaStream_t, the trainer's
 * stream that reads input_x) before this call -- an event recorded on it here,
 * waited on by the loader's copy -- so queued kernels still reading the previous
 * batch are never overwritten.  tm_loader_send uses the legacy default stream
 * (NULL), which covers work on blocking streams only. */
int tm_loader_send_after(tm_loader* loader, int kind, const char* filename, void* stream);
int tm_loader_send(tm_loader* loader, int kind, const char* filename);
/* Block until the next batch is in input_x (timeout_ms < 0: forever).
 * TM_E_IO / TM_E_CUDA / TM_E_ARG (protocol) if the loader failed;
 * TM_E_TIMEOUT; TM_E_STATE if the loader exited without a batch. */
int tm_loader_wait(tm_loader* loader, int64_t timeout_ms);
/* Send STOP, join the thread, free everything. */
int tm_loader_destroy(tm_loader* loader);

/* Synchronise `stream`, then return the most severe sticky status
 * (TM_E_TIMEOUT > TM_E_OVERFLOW16 > TM_E_NONFINITE > TM_OK) and clear it.
 * `bits` (optional) receives the TM_BIT_* mask.  The clear is enqueued on
 * `stream` and waited for before the call returns, so a bit set by any later
 * launch (on any stream) survives it. */
int tm_exchange_status(void* stream, uint32_t* bits);

/* Layout of the current exchanger (for tests and the bench). */
int tm_layout(tm_layout_info* out);

/* Select the data path (tm_path) for later exchanges of this exchanger.
 * TM_E_ARG for TM_PATH_DIRECT unless nlocal == size; TM_E_STATE before init. */
int tm_set_path(int path);

/* Select the allgather mode (tm_allgather) of later staged exchanges.  Every
 * rank must select the same mode before the same exchange.  TM_E_ARG for an
 * unknown mode; TM_E_NCCL for TM_AG_NCCL without a communicator; TM_E_STATE
 * before init. */
int tm_set_allgather(int mode);

/* Diagnostics: the staged kernels write %globaltimer (ns) of every CTA at its
 * phase boundaries into dev_buf[cta*8 + slot] (slot 0 start, 1 pre-cast done,
 * 2 READY acquired, 3 reduce-scatter done, 4 REDUCED acquired, 5 end; the
 * warp-specialised kernel overlaps pre-cast and reduce-scatter and writes only
 * 0, 3, 4, 5).  capacity in uint64 slots (>= nlocal*C*8, else ignored); NULL
 * disables. */
int tm_set_phase_log(uint64_t* dev_buf, int64_t capacity);

/* CTA budget of range (bucket) exchanges, per rank (0 = none, the default;
 * TM_RANGE_CTAS at init sets it too): a bucket exchanged while backward still
 * runs should occupy few SMs.  Staged path: at most `ctas` CTAs per rank (every
 * rank must set the same budget).  Direct path: the register kernel (no shared
 * memory, so its CTAs can share SMs with a GEMM's) on at most `ctas` CTAs.
 * Full exchanges (tm_exchange / tm_exchange_group) are not affected. */
int tm_set_range_ctas(int ctas);

/* Barrier spin timeout in nanoseconds (default 10 s; 0 restores default). */
int tm_set_timeout_ns(uint64_t ns);

/* Release everything; safe to call twice. */
int tm_exchange_finalize(void);

const char* tm_strerror(int status);

/* Test hook: the exact device rounding the ASA16 path uses (cvt.rn.f16.f32),
 * applied elementwise: out16[i] = rn16(in[i]) as binary16 bit patterns. */
int tm_cast_rn16(const float* in, uint16_t* out16, int64_t n, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* TM_H_ */
