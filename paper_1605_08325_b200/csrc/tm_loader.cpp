// The parallel loading process of Theano-MPI (Algorithm 1),
// B200-native: a native loader thread per training process (instead of an MPI
// Spawn'ed Python child, L359-364) reads batch files into pinned host memory,
// copies the RAW uint8 batch to the GPU on its own stream (4x fewer PCIe bytes
// than the preprocessed fp32 batch), runs the mean-subtract / crop / mirror
// kernel there (tm_loader_kernels.cu) into gpudata_x, and hands the batch to the
// trainer's input_x at the synchronisation point of Alg. 1.
//
// State machine (Alg. 1, line numbers of PAPER.md):
//   outer: receive mode (L330); "stop" -> exit (L331-332); else mode = recv.
//          receive the first filename (L336).
//   inner: load file into hostdata_x (L339), H2D + subtract mean + crop/mirror
//          into gpudata_x (L340-342, on the GPU), then wait for the next control
//          message (L343).  stop/train/val -> leave the inner loop (L344-345)
//          and treat that message as the next outer-loop message (reading
//          Q20: Alg. 1 would otherwise receive a second, unsent mode); else it is
//          the next filename (L347): copy gpudata_x -> input_x (L350),
//          synchronise (L351), notify the trainer (L352).
//
// Crop / mirror (Alg. 1 leaves the geometry open): train mode draws a
// crop offset in [0, h-ch] x [0, w-cw] and a mirror bit per example from
// splitmix64 of (seed, file counter, example); val mode takes the centre crop,
// no mirror.  The oracle implements the same counter-based generator.

#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <fcntl.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <deque>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "tm.h"
#include "tm_internal.h"

struct tm_loader {
  tm_loader_config cfg;
  float* input_x = nullptr;  // trainer-owned (device)
  // loader-owned
  uint8_t* host_raw = nullptr;   // hostdata_x (pinned)
  uint8_t* dev_raw = nullptr;
  float* dev_mean = nullptr;
  float* gpudata = nullptr;      // gpudata_x
  int32_t* host_crop = nullptr;  // pinned [n][3]
  int32_t* dev_crop = nullptr;
  cudaStream_t stream = nullptr;
  uint64_t file_counter = 0;

  std::thread th;
  std::mutex mu;
  std::condition_variable cv_msg, cv_ready;
  struct Msg {
    int kind;
    std::string file;
    cudaEvent_t after;  // FILE: the trainer's work that reads input_x (null = none)
  };
  std::deque<Msg> q;
  uint64_t delivered = 0, consumed = 0;
  int error = TM_OK;
  bool exited = false;
};

namespace {

uint64_t splitmix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// Crop offsets / mirror flags of one file (documented in tm.h).
void crop_params(const tm_loader_config& c, int mode, uint64_t file_counter, int32_t* out) {
  for (int b = 0; b < c.n; ++b) {
    if (mode == TM_LOADER_TRAIN) {
      const uint64_t z = splitmix64(c.seed ^ splitmix64((file_counter << 32) | (uint64_t)b));
      out[3 * b] = (int32_t)(z % (uint64_t)(c.h - c.crop_h + 1));
      out[3 * b + 1] = (int32_t)((z >> 20) % (uint64_t)(c.w - c.crop_w + 1));
      out[3 * b + 2] = (int32_t)((z >> 40) & 1);
    } else {
      out[3 * b] = (c.h - c.crop_h) / 2;
      out[3 * b + 1] = (c.w - c.crop_w) / 2;
      out[3 * b + 2] = 0;
    }
  }
}

// Alg. 1: load the file into hostdata_x and ship it to the GPU.  The
// payload is read in kChunks pieces by several threads (pread into the pinned
// buffer: one thread copying out of the page cache does ~10 GB/s), and each
// piece's H2D copy is issued, in order, as soon as it is in: reading and PCIe
// overlap.
int read_and_upload(tm_loader* L, const std::string& path) {
  FILE* f = fopen(path.c_str(), "rb");
  if (!f) return TM_E_IO;
  char magic[4];
  uint32_t dims[4];
  const bool ok = fread(magic, 1, 4, f) == 4 && memcmp(magic, "PXB1", 4) == 0 &&
                  fread(dims, 4, 4, f) == 4;
  fclose(f);
  const tm_loader_config& c = L->cfg;
  if (!ok || (int)dims[0] != c.n || (int)dims[1] != c.c || (int)dims[2] != c.h || (int)dims[3] != c.w)
    return TM_E_IO;
  const size_t bytes = (size_t)c.n * c.c * c.h * c.w;
  const int fd = open(path.c_str(), O_RDONLY);
  if (fd < 0) return TM_E_IO;
  constexpr int kChunks = 8;
  const off_t hdr = 4 + 4 * 4;
  const unsigned hw = std::thread::hardware_concurrency();
  const int nthr = (int)std::max<size_t>(1, std::min<size_t>({(size_t)4, hw ? (size_t)hw : 1, bytes >> 20}));
  std::atomic<int> next{0};
  std::mutex mu;
  std::condition_variable cv;
  std::vector<int> state(kChunks, 0);  // 0 pending, 1 read, -1 failed
  auto range = [&](int i, size_t& lo, size_t& hi) {
    lo = bytes * i / kChunks;
    hi = bytes * (i + 1) / kChunks;
  };
  std::vector<std::thread> ts;
  for (int t = 0; t < nthr; ++t) {
    ts.emplace_back([&] {
      for (int i = next++; i < kChunks; i = next++) {
        size_t lo, hi;
        range(i, lo, hi);
        size_t done = lo;
        while (done < hi) {
          const ssize_t r = pread(fd, L->host_raw + done, hi - done, hdr + (off_t)done);
          if (r <= 0) break;
          done += (size_t)r;
        }
        std::lock_guard<std::mutex> lk(mu);
        state[i] = done == hi ? 1 : -1;
        cv.notify_all();
      }
    });
  }
  int rc = TM_OK;
  for (int i = 0; i < kChunks && rc == TM_OK; ++i) {
    {
      std::unique_lock<std::mutex> lk(mu);
      cv.wait(lk, [&] { return state[i] != 0; });
      if (state[i] < 0) rc = TM_E_IO;
    }
    if (rc != TM_OK) break;
    size_t lo, hi;
    range(i, lo, hi);
    if (cudaMemcpyAsync(L->dev_raw + lo, L->host_raw + lo, hi - lo, cudaMemcpyHostToDevice, L->stream) !=
        cudaSuccess)
      rc = TM_E_CUDA;
  }
  for (auto& th : ts) th.join();
  close(fd);
  return rc;
}

// Alg. 1: load, H2D, preprocess into gpudata_x (synchronous on the
// loader's stream: the host buffer is reused for the next file).
int load_and_preprocess(tm_loader* L, int mode, const std::string& path) {
  int rc = read_and_upload(L, path);
  if (rc != TM_OK) {
    cudaStreamSynchronize(L->stream);  // no copy may still read host_raw
    return rc;
  }
  const tm_loader_config& c = L->cfg;
  crop_params(c, mode, L->file_counter++, L->host_crop);
  if (cudaMemcpyAsync(L->dev_crop, L->host_crop, (size_t)c.n * 3 * 4, cudaMemcpyHostToDevice, L->stream) !=
          cudaSuccess ||
      tmx::launch_preprocess(L->dev_raw, L->dev_mean, L->dev_crop, L->gpudata, c.n, c.c, c.h, c.w,
                             c.crop_h, c.crop_w, L->stream) != cudaSuccess ||
      cudaStreamSynchronize(L->stream) != cudaSuccess)
    return TM_E_CUDA;
  return TM_OK;
}

tm_loader::Msg recv(tm_loader* L) {
  std::unique_lock<std::mutex> lk(L->mu);
  L->cv_msg.wait(lk, [&] { return !L->q.empty(); });
  auto m = L->q.front();
  L->q.pop_front();
  return m;
}

void drop_event(tm_loader::Msg& m) {
  if (m.after) cudaEventDestroy(m.after);
  m.after = nullptr;
}

void fail(tm_loader* L, int rc) {
  std::lock_guard<std::mutex> lk(L->mu);
  if (L->error == TM_OK) L->error = rc;
  L->cv_ready.notify_all();
}

void loader_main(tm_loader* L) {
  cudaSetDevice(L->cfg.device);
  tm_loader::Msg msg = recv(L);  // L330
  for (;;) {
    drop_event(msg);  // nothing to order before a mode message or the first file
    if (msg.kind == TM_LOADER_STOP) break;  // L331-332
    if (msg.kind != TM_LOADER_TRAIN && msg.kind != TM_LOADER_VAL) {
      fail(L, TM_E_ARG);  // protocol violation: a filename where a mode was due
      break;
    }
    const int mode = msg.kind;  // L334
    msg = recv(L);              // L336: the first filename
    drop_event(msg);
    if (msg.kind != TM_LOADER_FILE) {
      fail(L, TM_E_ARG);
      break;
    }
    std::string filename = msg.file;
    bool stop_outer = false;
    for (;;) {
      const int rc = load_and_preprocess(L, mode, filename);  // L339-342
      if (rc != TM_OK) {
        fail(L, rc);
        stop_outer = true;
        break;
      }
      msg = recv(L);  // L343: wait for training on the last input_x
      if (msg.kind != TM_LOADER_FILE) break;  // L344-345 (msg feeds the outer loop)
      filename = msg.file;                    // L347
      const tm_loader_config& c = L->cfg;
      const size_t out_bytes = (size_t)c.n * c.c * c.crop_h * c.crop_w * sizeof(float);
      // The trainer's kernels that read input_x may still be queued on its stream
      // when the FILE message arrives: the copy waits for the event recorded on
      // that stream at send time, so it cannot overwrite input_x under them.
      const bool ok_wait = !msg.after || cudaStreamWaitEvent(L->stream, msg.after, 0) == cudaSuccess;
      const bool ok = ok_wait &&
                      cudaMemcpyAsync(L->input_x, L->gpudata, out_bytes, cudaMemcpyDeviceToDevice,
                                      L->stream) == cudaSuccess &&
                      cudaStreamSynchronize(L->stream) == cudaSuccess;  // L350-351
      drop_event(msg);
      if (!ok) {
        fail(L, TM_E_CUDA);
        stop_outer = true;
        break;
      }
      {
        std::lock_guard<std::mutex> lk(L->mu);  // L352: notify the trainer
        ++L->delivered;
      }
      L->cv_ready.notify_all();
    }
    if (stop_outer) break;
  }
  drop_event(msg);
  std::lock_guard<std::mutex> lk(L->mu);
  L->exited = true;
  for (auto& m : L->q) drop_event(m);
  L->cv_ready.notify_all();
}

void free_loader(tm_loader* L) {
  if (L->stream) cudaStreamDestroy(L->stream);
  if (L->host_raw) cudaFreeHost(L->host_raw);
  if (L->host_crop) cudaFreeHost(L->host_crop);
  if (L->dev_raw) cudaFree(L->dev_raw);
  if (L->dev_mean) cudaFree(L->dev_mean);
  if (L->gpudata) cudaFree(L->gpudata);
  if (L->dev_crop) cudaFree(L->dev_crop);
  delete L;
}

}  // namespace

extern "C" {

int tm_loader_create(const tm_loader_config* cfg, float* input_x, tm_loader** out) {
  if (!cfg || !input_x || !out || !cfg->mean) return TM_E_ARG;
  const tm_loader_config& c = *cfg;
  if (c.n < 1 || c.c < 1 || c.h < 1 || c.w < 1 || c.crop_h < 1 || c.crop_w < 1 || c.crop_h > c.h ||
      c.crop_w > c.w)
    return TM_E_ARG;
  if (cudaSetDevice(c.device) != cudaSuccess) return TM_E_CUDA;
  tm_loader* L = new tm_loader();
  L->cfg = c;
  L->cfg.mean = nullptr;  // host copy not retained
  L->input_x = input_x;
  const size_t raw = (size_t)c.n * c.c * c.h * c.w;
  const size_t img = (size_t)c.c * c.h * c.w;
  const size_t outn = (size_t)c.n * c.c * c.crop_h * c.crop_w;
  if (cudaHostAlloc(reinterpret_cast<void**>(&L->host_raw), raw, cudaHostAllocDefault) != cudaSuccess ||
      cudaHostAlloc(reinterpret_cast<void**>(&L->host_crop), (size_t)c.n * 3 * 4, cudaHostAllocDefault) !=
          cudaSuccess ||
      cudaMalloc(reinterpret_cast<void**>(&L->dev_raw), raw) != cudaSuccess ||
      cudaMalloc(reinterpret_cast<void**>(&L->dev_mean), img * 4) != cudaSuccess ||
      cudaMalloc(reinterpret_cast<void**>(&L->gpudata), outn * 4) != cudaSuccess ||
      cudaMalloc(reinterpret_cast<void**>(&L->dev_crop), (size_t)c.n * 3 * 4) != cudaSuccess ||
      cudaStreamCreateWithFlags(&L->stream, cudaStreamNonBlocking) != cudaSuccess ||
      cudaMemcpy(L->dev_mean, cfg->mean, img * 4, cudaMemcpyHostToDevice) != cudaSuccess ||
      // a pageable-memory cudaMemcpy may return before its DMA lands; the loader's
      // stream is non-blocking, so wait before its first preprocess kernel
      cudaDeviceSynchronize() != cudaSuccess) {
    free_loader(L);
    return TM_E_CUDA;
  }
  L->th = std::thread(loader_main, L);
  *out = L;
  return TM_OK;
}

int tm_loader_send_after(tm_loader* L, int kind, const char* filename, void* stream) {
  if (!L) return TM_E_ARG;
  if (kind < TM_LOADER_TRAIN || kind > TM_LOADER_FILE) return TM_E_ARG;
  if (kind == TM_LOADER_FILE && !filename) return TM_E_ARG;
  cudaEvent_t ev = nullptr;
  if (kind == TM_LOADER_FILE) {  // the trainer's work enqueued so far on `stream`
    int prev = 0;  // the caller's current device is restored below
    if (cudaGetDevice(&prev) != cudaSuccess || cudaSetDevice(L->cfg.device) != cudaSuccess) return TM_E_CUDA;
    bool ok = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) == cudaSuccess;
    if (ok && cudaEventRecord(ev, static_cast<cudaStream_t>(stream)) != cudaSuccess) {
      cudaEventDestroy(ev);
      ok = false;
    }
    cudaSetDevice(prev);
    if (!ok) return TM_E_CUDA;
  }
  {
    std::lock_guard<std::mutex> lk(L->mu);
    L->q.push_back({kind, kind == TM_LOADER_FILE ? std::string(filename) : std::string(), ev});
  }
  L->cv_msg.notify_all();
  return TM_OK;
}

int tm_loader_send(tm_loader* L, int kind, const char* filename) {
  return tm_loader_send_after(L, kind, filename, nullptr);  // legacy default stream
}

int tm_loader_wait(tm_loader* L, int64_t timeout_ms) {
  if (!L) return TM_E_ARG;
  std::unique_lock<std::mutex> lk(L->mu);
  auto pred = [&] { return L->delivered > L->consumed || L->error != TM_OK || L->exited; };
  if (timeout_ms < 0) {
    L->cv_ready.wait(lk, pred);
  } else if (!L->cv_ready.wait_for(lk, std::chrono::milliseconds(timeout_ms), pred)) {
    return TM_E_TIMEOUT;
  }
  if (L->delivered > L->consumed) {
    ++L->consumed;
    return TM_OK;
  }
  return L->error != TM_OK ? L->error : TM_E_STATE;
}

int tm_loader_destroy(tm_loader* L) {
  if (!L) return TM_OK;
  {
    std::lock_guard<std::mutex> lk(L->mu);
    L->q.push_back({TM_LOADER_STOP, std::string(), nullptr});
  }
  L->cv_msg.notify_all();
  if (L->th.joinable()) L->th.join();
  free_loader(L);
  return TM_OK;
}

}  // extern "C"
