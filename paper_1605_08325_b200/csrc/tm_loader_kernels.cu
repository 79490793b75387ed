// Preprocessing kernel of the parallel loading process (PAPER Alg. 1):
// "hostdata_x = hostdata_x - image_mean; crop and mirror hostdata_x according to
// mode".  B200-native: the raw uint8 batch crosses PCIe (4x fewer bytes than the
// fp32 result) and the arithmetic runs here, one thread per output element:
//
//   out[b][ch][y][x] = fl(float(raw[b][ch][oy+y][ox+xs]) - mean[ch][oy+y][ox+xs]),
//   xs = mirror_b ? cw - 1 - x : x
//
// (mean subtracted from the full image first, then the crop window is taken and
// mirrored: the order of Alg. 1; one fp32 rounding).  Crop offsets
// and mirror flags per example are computed on the host (tm_loader.cpp) and
// passed in.

#include <stdint.h>

#include "tm_internal.h"

namespace tmx {
namespace {

__global__ void __launch_bounds__(256)
preprocess_kernel(const uint8_t* __restrict__ raw, const float* __restrict__ mean,
                  const int32_t* __restrict__ crop, float* __restrict__ out, int n, int c, int h,
                  int w, int ch, int cw) {
  const int64_t total = (int64_t)n * c * ch * cw;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += stride) {
    const int x = (int)(i % cw);
    int64_t t = i / cw;
    const int y = (int)(t % ch);
    t /= ch;
    const int k = (int)(t % c);
    const int b = (int)(t / c);
    const int oy = crop[3 * b], ox = crop[3 * b + 1], mir = crop[3 * b + 2];
    const int xs = mir ? cw - 1 - x : x;
    const int64_t src = (((int64_t)b * c + k) * h + (oy + y)) * w + (ox + xs);
    const int64_t msrc = ((int64_t)k * h + (oy + y)) * w + (ox + xs);
    out[i] = __fsub_rn((float)raw[src], mean[msrc]);
  }
}

}  // namespace

cudaError_t launch_preprocess(const uint8_t* raw, const float* mean, const int32_t* crop, float* out,
                              int n, int c, int h, int w, int ch, int cw, cudaStream_t s) {
  const int64_t total = (int64_t)n * c * ch * cw;
  int dev = 0, sms = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t want = (total + 255) / 256;
  const int grid = (int)(want < 8LL * sms ? (want > 0 ? want : 1) : 8LL * sms);
  preprocess_kernel<<<grid, 256, 0, s>>>(raw, mean, crop, out, n, c, h, w, ch, cw);
  return cudaGetLastError();
}

}  // namespace tmx
