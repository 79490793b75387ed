// HBM ceiling probe (diagnostics, not part of libtm.so): what read-only,
// write-only and 1:1 read/write (copy) streams reach on this B200, for the
// access styles the exchange kernels use -- 16-byte register loads/stores and
// 1-D bulk copies (cp.async.bulk) through a shared-memory ring.  The headline
// direct kernel is a 1:1 read/write stream (8 B per element per rank), so the
// copy figures are its ceiling.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/hbm_probe tools/hbm_probe.cu
//   /tmp/hbm_probe [GiB per buffer, default 2]
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#define CK(x)                                                                        \
  do {                                                                               \
    cudaError_t e_ = (x);                                                            \
    if (e_ != cudaSuccess) {                                                         \
      fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_));     \
      exit(1);                                                                       \
    }                                                                                \
  } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// ---- register path ----------------------------------------------------------
__global__ void read_ldg(const float4* __restrict__ a, size_t n, float* out) {
  float4 acc = make_float4(0, 0, 0, 0);
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    float4 v = __ldcs(a + i);
    acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
  }
  if (acc.x + acc.y + acc.z + acc.w == 1234.5f) *out = acc.x;
}
__global__ void write_stg(float4* __restrict__ a, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    __stcs(a + i, make_float4(1, 2, 3, 4));
}
template <int U>
__global__ void copy_ldg(const float4* __restrict__ a, float4* __restrict__ b, size_t n) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  for (; i + (U - 1) * stride < n; i += U * stride) {
    float4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = __ldcs(a + i + u * stride);
#pragma unroll
    for (int u = 0; u < U; ++u) __stcs(b + i + u * stride, v[u]);
  }
  for (; i < n; i += stride) __stcs(b + i, __ldcs(a + i));
}

// ---- bulk-copy path: thread 0 streams tiles through an S-deep ring ------------
template <int TILE_BYTES, int S>
__global__ void __launch_bounds__(128, 1) copy_bulk(const char* __restrict__ a, char* __restrict__ b, size_t ntiles) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) uint64_t full[S];
  if (threadIdx.x != 0) return;
  for (int s = 0; s < S; ++s)
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&full[s])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  size_t t0 = blockIdx.x;
  const size_t step = gridDim.x;
  auto issue = [&](size_t i, size_t t) {
    const int s = (int)(i % S);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&full[s])), "r"(TILE_BYTES)
                 : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(smem + (size_t)s * TILE_BYTES)),
                 "l"(a + t * TILE_BYTES), "r"(TILE_BYTES), "r"(smem_u32(&full[s]))
                 : "memory");
  };
  size_t nmine = t0 < ntiles ? (ntiles - t0 + step - 1) / step : 0;
  for (size_t i = 0; i < (size_t)S && i < nmine; ++i) issue(i, t0 + i * step);
  for (size_t i = 0; i < nmine; ++i) {
    const int s = (int)(i % S);
    const uint32_t par = (uint32_t)((i / S) & 1);
    asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(
                     smem_u32(&full[s])),
                 "r"(par)
                 : "memory");
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(b + (t0 + i * step) * TILE_BYTES),
                 "r"(smem_u32(smem + (size_t)s * TILE_BYTES)), "r"(TILE_BYTES)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    if (i + S < nmine) {
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // slot s read out before reuse
      issue(i + S, t0 + (i + S) * step);
    }
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

template <class F>
float time_ms(F f, int reps) {
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  f();
  CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    CK(cudaEventRecord(e0));
    f();
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    if (ms < best) best = ms;
  }
  return best;
}

template <int TB, int S>
void run_bulk(const char* a, char* b, size_t bytes, int sms, int per_sm) {
  const size_t ntiles = bytes / TB;
  const int smem = TB * S;
  CK(cudaFuncSetAttribute(copy_bulk<TB, S>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  const int grid = sms * per_sm;
  float ms = time_ms([&] { copy_bulk<TB, S><<<grid, 128, smem>>>(a, b, ntiles); }, 10);
  CK(cudaGetLastError());
  printf("copy bulk tile %6d B x %d stages, %d CTA/SM: %8.1f GB/s (read+write)\n", TB, S, per_sm,
         2.0 * ntiles * TB / (ms * 1e-3) / 1e9);
}

int main(int argc, char** argv) {
  const double gib = argc > 1 ? atof(argv[1]) : 2.0;
  const size_t bytes = (size_t)(gib * (1ull << 30)) / 65536 * 65536;
  int dev = 0, sms = 0;
  CK(cudaGetDevice(&dev));
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  char *a, *b;
  float* out;
  CK(cudaMalloc(&a, bytes));
  CK(cudaMalloc(&b, bytes));
  CK(cudaMalloc(&out, 4));
  CK(cudaMemset(a, 1, bytes));
  CK(cudaMemset(b, 2, bytes));
  CK(cudaDeviceSynchronize());
  const size_t n4 = bytes / 16;
  printf("buffers: 2 x %.2f GiB, %d SMs\n", bytes / double(1ull << 30), sms);
  for (int per_sm : {2, 4, 8}) {
    float ms = time_ms([&] { read_ldg<<<sms * per_sm, 512>>>((const float4*)a, n4, out); }, 10);
    printf("read  ldg.128, %d x 512 thr/SM:           %8.1f GB/s\n", per_sm, bytes / (ms * 1e-3) / 1e9);
    ms = time_ms([&] { write_stg<<<sms * per_sm, 512>>>((float4*)b, n4); }, 10);
    printf("write stg.128, %d x 512 thr/SM:           %8.1f GB/s\n", per_sm, bytes / (ms * 1e-3) / 1e9);
  }
  for (int per_sm : {2, 4}) {
    float ms = time_ms([&] { copy_ldg<4><<<sms * per_sm, 512>>>((const float4*)a, (float4*)b, n4); }, 10);
    printf("copy ldg/stg x4 unroll, %d x 512 thr/SM:   %8.1f GB/s (read+write)\n", per_sm, 2.0 * bytes / (ms * 1e-3) / 1e9);
    ms = time_ms([&] { copy_ldg<8><<<sms * per_sm, 512>>>((const float4*)a, (float4*)b, n4); }, 10);
    printf("copy ldg/stg x8 unroll, %d x 512 thr/SM:   %8.1f GB/s (read+write)\n", per_sm, 2.0 * bytes / (ms * 1e-3) / 1e9);
  }
  float ms = time_ms([&] { CK(cudaMemcpyAsync(b, a, bytes, cudaMemcpyDeviceToDevice)); }, 10);
  printf("cudaMemcpy D2D:                            %8.1f GB/s (read+write)\n", 2.0 * bytes / (ms * 1e-3) / 1e9);
  run_bulk<8192, 8>(a, b, bytes, sms, 1);
  run_bulk<16384, 8>(a, b, bytes, sms, 1);
  run_bulk<32768, 6>(a, b, bytes, sms, 1);
  run_bulk<16384, 6>(a, b, bytes, sms, 2);
  run_bulk<65536, 3>(a, b, bytes, sms, 1);
  return 0;
}
