// NVLink evidence on a one-GPU box: a multicast object (NVLS) with ONE member
// device.  A store to the multicast address leaves the SM through the GPU's
// NVLink ports, is replicated by the NVSwitch to the group's members (here the
// GPU itself) and lands in its own HBM; a multimem.ld_reduce is served by the
// switch the same way.  So the bandwidth of those kernels is a measured bound
// of the GPU <-> NVSwitch path on this box, and ncu's nvltx / nvlrx counters of
// them show the bytes crossing the links -- the links the exchange's peer loads
// use on an 8-GPU box (roofline 900 GB/s per direction).
// Diagnostics tool only (not the exchange's data path; every value it moves is
// a plain copy, checked bitwise on the host).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o nvls_probe tools/nvls_probe.cu -lcuda
//   ./nvls_probe [MiB=1024] [reps=20]
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include <algorithm>
#include <vector>

#define CK(x)                                                                                  \
  do {                                                                                         \
    CUresult r_ = (x);                                                                         \
    if (r_ != CUDA_SUCCESS) {                                                                  \
      const char* s_ = nullptr;                                                                \
      cuGetErrorString(r_, &s_);                                                               \
      printf("{\"probe\": \"nvls\", \"error\": \"%s -> %d %s\"}\n", #x, (int)r_, s_ ? s_ : ""); \
      return 1;                                                                                \
    }                                                                                          \
  } while (0)
#define CR(x)                                                                                    \
  do {                                                                                           \
    cudaError_t e_ = (x);                                                                        \
    if (e_ != cudaSuccess) {                                                                     \
      printf("{\"probe\": \"nvls\", \"error\": \"%s -> %s\"}\n", #x, cudaGetErrorString(e_));   \
      return 1;                                                                                  \
    }                                                                                            \
  } while (0)

// value of element i: distinct per element, exact in fp32
__device__ __forceinline__ float val(int64_t i, float salt) { return (float)(i & 0xFFFFF) + salt; }

__global__ void mc_store(float* mc, int64_t n4, float salt) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n4; v += stride) {
    const int64_t i = v * 4;
    asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(mc + i),
                 "f"(val(i, salt)), "f"(val(i + 1, salt)), "f"(val(i + 2, salt)), "f"(val(i + 3, salt))
                 : "memory");
  }
}

__global__ void mc_ld_reduce(const float* mc, float* out, int64_t n4) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  float acc = 0.f;
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n4; v += stride) {
    float a, b, c, d;
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(a), "=f"(b), "=f"(c), "=f"(d)
                 : "l"(mc + v * 4)
                 : "memory");
    acc += a + b + c + d;
  }
  if (acc == -1.0f) out[0] = acc;  // keep the loads
}

// unicast comparison: plain 16-byte stores / loads to the same physical memory (HBM)
__global__ void uc_store(float* p, int64_t n4, float salt) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n4; v += stride) {
    const int64_t i = v * 4;
    reinterpret_cast<float4*>(p)[v] = make_float4(val(i, salt), val(i + 1, salt), val(i + 2, salt), val(i + 3, salt));
  }
}
__global__ void uc_load(const float* p, float* out, int64_t n4) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  float acc = 0.f;
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n4; v += stride) {
    const float4 t = __ldcs(reinterpret_cast<const float4*>(p) + v);
    acc += t.x + t.y + t.z + t.w;
  }
  if (acc == -1.0f) out[0] = acc;
}

int main(int argc, char** argv) {
  const int64_t mib = argc > 1 ? atoll(argv[1]) : 1024;
  const int reps = argc > 2 ? atoi(argv[2]) : 20;
  CR(cudaSetDevice(0));
  CR(cudaFree(0));
  CUdevice dev;
  CK(cuDeviceGet(&dev, 0));
  int mc_ok = 0, nsm = 0;
  CK(cuDeviceGetAttribute(&mc_ok, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev));
  CK(cuDeviceGetAttribute(&nsm, CU_DEVICE_ATTRIBUTE_MULTIPROCESSOR_COUNT, dev));
  if (!mc_ok) {
    printf("{\"probe\": \"nvls\", \"multicast_supported\": 0}\n");
    return 0;
  }
  // the handle types the driver accepts for a one-member group vary (a fabric
  // handle needs IMEX): try them in turn, report each refusal
  const int htypes[] = {CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, CU_MEM_HANDLE_TYPE_NONE,
                        CU_MEM_HANDLE_TYPE_FABRIC};
  CUmulticastObjectProp mp = {};
  CUmemGenericAllocationHandle mc;
  size_t gran = 0, gran_min = 0, size = 0;
  bool made = false;
  const int ndev_try = getenv("NVLS_NDEV") ? atoi(getenv("NVLS_NDEV")) : 1;
  for (int ht : htypes) {
    mp = {};
    mp.numDevices = ndev_try;
    mp.handleTypes = (unsigned long long)ht;
    mp.size = (size_t)mib << 20;
    CUresult r = cuMulticastGetGranularity(&gran, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED);
    if (r == CUDA_SUCCESS) r = cuMulticastGetGranularity(&gran_min, &mp, CU_MULTICAST_GRANULARITY_MINIMUM);
    if (r == CUDA_SUCCESS) {
      size = (mp.size + gran - 1) / gran * gran;
      mp.size = size;
      r = cuMulticastCreate(&mc, &mp);
    }
    const char* es = nullptr;
    cuGetErrorString(r, &es);
    fprintf(stderr, "[nvls] handle type %d: granularity %zu / %zu, cuMulticastCreate -> %d %s\n", ht, gran,
            gran_min, (int)r, es ? es : "");
    if (r == CUDA_SUCCESS) {
      made = true;
      break;
    }
  }
  if (!made) {
    printf("{\"probe\": \"nvls\", \"multicast_supported\": 1, \"error\": \"cuMulticastCreate refused every handle type (stderr)\"}\n");
    return 1;
  }
  CK(cuMulticastAddDevice(mc, dev));
  CUmemAllocationProp ap = {};
  ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ap.location.id = 0;
  ap.requestedHandleTypes = (CUmemAllocationHandleType)mp.handleTypes;
  size_t pgran = 0;
  CK(cuMemGetAllocationGranularity(&pgran, &ap, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED));
  CUmemGenericAllocationHandle phys;
  CK(cuMemCreate(&phys, size, &ap, 0));
  CK(cuMulticastBindMem(mc, 0, phys, 0, size, 0));
  CUmemAccessDesc acc = {};
  acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  acc.location.id = 0;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  CUdeviceptr mcva = 0, ucva = 0;
  const size_t align = gran > pgran ? gran : pgran;
  CK(cuMemAddressReserve(&mcva, size, align, 0, 0));
  CK(cuMemMap(mcva, size, 0, mc, 0));
  CK(cuMemSetAccess(mcva, size, &acc, 1));
  CK(cuMemAddressReserve(&ucva, size, align, 0, 0));
  CK(cuMemMap(ucva, size, 0, phys, 0));
  CK(cuMemSetAccess(ucva, size, &acc, 1));

  float* mcp = reinterpret_cast<float*>(mcva);
  float* ucp = reinterpret_cast<float*>(ucva);
  float* sink = nullptr;
  CR(cudaMalloc(&sink, 16));
  const int64_t n = (int64_t)(size / 4), n4 = n / 4;
  const int grid = 4 * nsm, block = 256;
  cudaEvent_t e0, e1;
  CR(cudaEventCreate(&e0));
  CR(cudaEventCreate(&e1));

  auto time_it = [&](auto launch) -> double {  // median of reps, ms
    launch();
    launch();
    cudaDeviceSynchronize();
    std::vector<float> t;
    for (int r = 0; r < reps; ++r) {
      cudaEventRecord(e0);
      launch();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      t.push_back(ms);
    }
    std::sort(t.begin(), t.end());
    return t[t.size() / 2];
  };

  // correctness: a multicast store must land in the (unicast view of the) memory
  CR(cudaMemset(ucp, 0, size));
  mc_store<<<grid, block>>>(mcp, n4, 0.5f);
  CR(cudaDeviceSynchronize());
  std::vector<float> h(1 << 20);
  int64_t bad = 0, checked = 0;
  for (int64_t off : {(int64_t)0, n / 2, n - (int64_t)h.size()}) {
    CR(cudaMemcpy(h.data(), ucp + off, h.size() * 4, cudaMemcpyDeviceToHost));
    for (size_t j = 0; j < h.size(); ++j) {
      const int64_t i = off + (int64_t)j;
      const float want = (float)(i & 0xFFFFF) + 0.5f;
      bad += h[j] != want;
      ++checked;
    }
  }
  const double gb = (double)size / 1e9;
  const double t_mst = time_it([&] { mc_store<<<grid, block>>>(mcp, n4, 1.5f); });
  const double t_mld = time_it([&] { mc_ld_reduce<<<grid, block>>>(mcp, sink, n4); });
  const double t_ust = time_it([&] { uc_store<<<grid, block>>>(ucp, n4, 2.5f); });
  const double t_uld = time_it([&] { uc_load<<<grid, block>>>(ucp, sink, n4); });
  CR(cudaGetLastError());
  CR(cudaDeviceSynchronize());
  printf("{\"probe\": \"nvls\", \"multicast_supported\": 1, \"members\": 1, \"bytes\": %zu, "
         "\"granularity\": %zu, \"granularity_min\": %zu, \"grid\": %d, \"reps\": %d, "
         "\"store_check\": {\"checked\": %lld, \"bad\": %lld}, "
         "\"multimem_st_GBps\": %.1f, \"multimem_ld_reduce_GBps\": %.1f, "
         "\"unicast_st_GBps\": %.1f, \"unicast_ld_GBps\": %.1f, "
         "\"ms\": {\"multimem_st\": %.4f, \"multimem_ld_reduce\": %.4f, \"unicast_st\": %.4f, \"unicast_ld\": %.4f}}\n",
         size, gran, gran_min, grid, reps, (long long)checked, (long long)bad, gb / (t_mst * 1e-3),
         gb / (t_mld * 1e-3), gb / (t_ust * 1e-3), gb / (t_uld * 1e-3), t_mst, t_mld, t_ust, t_uld);
  cuMemUnmap(mcva, size);
  cuMemUnmap(ucva, size);
  cuMemAddressFree(mcva, size);
  cuMemAddressFree(ucva, size);
  cuMemRelease(phys);
  cuMemRelease(mc);
  return bad == 0 ? 0 : 2;
}
