// sm_100a staged exchange (tm_staged.cuh holds the kernels and the protocol
// notes): instantiation of the plain kernels, occupancy, and the launch.
#include "tm_staged.cuh"

namespace tmx {

// tm_staged_sgd.cu: the kernels with the BSP step fused into the pre-cast.
const void* pick_exchange_sgd(int k, bool w16, bool sys, int fl);


namespace {
// x[i] = widen(gather[i]) for i < P: 8 elements (16 bytes of fp16) per thread-step.
__global__ void __launch_bounds__(kThreads)
widen16_kernel(const uint4* __restrict__ g, float* __restrict__ x, int64_t P) {
  const int64_t stride = (int64_t)gridDim.x * kThreads;
  const int64_t n8 = P / 8;
  for (int64_t v = (int64_t)blockIdx.x * kThreads + threadIdx.x; v < n8; v += stride) {
    float f[8];
    Unit<true>::decode(__ldcs(g + v), f);
    Unit<true>::store_dst(x + v * 8, f);
  }
  const int64_t i = n8 * 8 + (int64_t)blockIdx.x * kThreads + threadIdx.x;
  if (blockIdx.x == 0 && i < P)
    x[i] = __half2float(reinterpret_cast<const __half*>(g)[i]);
}
}  // namespace

cudaError_t launch_widen16(const void* gather, float* x, int64_t P, cudaStream_t s) {
  widen16_kernel<<<streaming_grid(P / 8 + 8), kThreads, 0, s>>>(static_cast<const uint4*>(gather), x, P);
  return cudaGetLastError();
}

int exchange_max_ctas(int device, bool wire16, int k, int fl) {
  // every instantiation a launch of this flavour may use: plain and with the
  // fused BSP step (its own register allocation), GPU and system scope -- the
  // cooperative launch needs all of the grid co-resident for any of them
  int per_sm_min = -1;
  for (int sgd = 0; sgd < 2; ++sgd)
    for (int sys = 0; sys < 2; ++sys) {
      const void* fn = sgd ? pick_exchange_sgd(k, wire16, sys != 0, fl) : pick_exchange<false>(k, wire16, sys != 0, fl);
      if (!fn) return 0;
      if (prepare(fn, fl) != cudaSuccess) return 0;
      int per_sm = 0;
      if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, flavour_threads(fl), flavour_smem(fl)) !=
          cudaSuccess)
        return 0;
      per_sm_min = per_sm_min < 0 ? per_sm : std::min(per_sm_min, per_sm);
    }
  return per_sm_min * sm_count(device);
}

cudaError_t launch_exchange(const ExchangeArgs& a, int nlocal, bool wire16, int fl, cudaStream_t s) {
  // System-scope flags only when some peer rank lives in another process
  // (another GPU, over NVLink); a single-process group syncs at GPU scope.
  const bool sys = nlocal != a.k;
  const void* fn = a.sgd ? pick_exchange_sgd(a.k, wire16, sys, fl) : pick_exchange<false>(a.k, wire16, sys, fl);
  if (!fn) return cudaErrorInvalidValue;
  cudaError_t e = prepare(fn, fl);
  if (e != cudaSuccess) return e;
  void* params[] = {const_cast<ExchangeArgs*>(&a)};
  // Cooperative launch: guarantees every CTA is co-resident, which the
  // per-CTA flag barriers need when several ranks share this device.
  e = cudaLaunchCooperativeKernel(fn, dim3(nlocal * a.C), dim3(flavour_threads(fl)), params,
                                  flavour_smem(fl), s);
  if (e != cudaSuccess) cudaGetLastError();  // returned here; do not leave it for the next launch's check
  return e;
}

}  // namespace tmx
