/* Plain-C use of the boundary (include/tm.h) without Python or torch: k ranks in
 * one process on one GPU (a single-process group), ASA16 exchange of a ragged P,
 * result compared with a host recomputation of the same definition (the
 * documented arithmetic of tm.h, using the C library's fp16 conversion).
 *
*   gcc -O2 -std=c11 -I include -I /usr/local/cuda/include examples/exchange_c.c -L paper_1605_08325_b200 -ltm \
 *       -L /usr/local/cuda/lib64 -lcudart -Wl,-rpath,$PWD/paper_1605_08325_b200 -o exchange_c
 */
#include <cuda_runtime_api.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "tm.h"

#define CHECK_TM(x)                                                        \
  do {                                                                     \
    int rc_ = (x);                                                         \
    if (rc_ != TM_OK) {                                                    \
      fprintf(stderr, "%s failed: %d (%s)\n", #x, rc_, tm_strerror(rc_)); \
      return 1;                                                            \
    }                                                                      \
  } while (0)

/* binary16 round trip with the C compiler's IEEE conversion (_Float16, RNE). */
static float rt16(float x) { return (float)(_Float16)x; }

int main(void) {
  const int k = 4;
  const int64_t P = 100003;
  float* host[4];
  float* dev[4];
  srand(1605);
  for (int r = 0; r < k; ++r) {
    host[r] = (float*)malloc(P * sizeof(float));
    for (int64_t i = 0; i < P; ++i) host[r][i] = ((float)rand() / RAND_MAX - 0.5f) * 0.02f;
    if (cudaMalloc((void**)&dev[r], P * sizeof(float)) != cudaSuccess) return 1;
    cudaMemcpy(dev[r], host[r], P * sizeof(float), cudaMemcpyHostToDevice);
  }
  tm_world world = {0, k, 0, k};
  CHECK_TM(tm_exchange_init(P, &world, TM_ASA16));
  CHECK_TM(tm_exchange_group(dev, k, NULL));
  uint32_t bits = 0;
  CHECK_TM(tm_exchange_status(NULL, &bits));
  float* out = (float*)malloc(P * sizeof(float));
  long bad = 0;
  for (int r = 0; r < k; ++r) {
    cudaMemcpy(out, dev[r], P * sizeof(float), cudaMemcpyDeviceToHost);
    for (int64_t i = 0; i < P; ++i) {
      volatile float s = rt16(host[0][i]);  /* volatile: one rounding per step */
      for (int j = 1; j < k; ++j) s = s + rt16(host[j][i]);
      volatile float a = s / (float)k;
      const float want = rt16(a);
      if (memcmp(&want, &out[i], 4) != 0) ++bad;
    }
  }
  tm_exchange_finalize();
  printf("exchange_c: k=%d P=%lld ASA16 mismatches=%ld status_bits=%u\n", k, (long long)P, bad, bits);
  return bad == 0 ? 0 : 2;
}
