/* c_abi_fill.c -- the drop-in boundary used from plain C (no Python, no torch).
 *
 * Draws this rank's window of a Shard(1) Uniform01 float32 tensor and a fused
 * dropout through include/sdrng.h, then checks every element against the
 * host Philox entry point (sdr_philox_block_host) using the reference's own
 * formulas: u = (w0 >> 8) * 2^-24 (rng.py:118-127) and keep <=> the 53-bit
 * u of (w1:w0) < ceil((1-p) 2^53) (rng.py:174-182, 238-242).
 *
 *   gcc -O2 -Iinclude -I/usr/local/cuda/include examples/c_abi_fill.c \
 *       -Lpaper_2509_07003_b200 -lsdrng -L/usr/local/cuda/lib64 -lcudart -o c_abi_fill
 */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <cuda_runtime_api.h>

#include "sdrng.h"

#define CHECK(x)                                                                  \
  do {                                                                            \
    int32_t st_ = (x);                                                            \
    if (st_ != SDR_OK) {                                                          \
      fprintf(stderr, "%s failed: %s (%s)\n", #x, sdr_strerror(st_), sdr_last_cuda_error()); \
      return 1;                                                                   \
    }                                                                             \
  } while (0)

int main(void) {
  /* global [6, 1000] float32, mesh of 4 ranks, Shard(1): rank 2 owns columns [500, 750) */
  const int64_t G0 = 6, G1 = 1000, c0 = 500, nc = 250;
  const uint64_t seed = 20240817, offset = 3, theta = 64;
  sdr_view v;
  memset(&v, 0, sizeof(v));
  v.ndim = 2;
  v.global_shape[0] = G0; v.global_shape[1] = G1;
  v.local_start[0] = 0;   v.local_start[1] = c0;
  v.local_len[0] = G0;    v.local_len[1] = nc;
  v.groups[0] = 1;        v.groups[1] = 1;
  sdr_rng r = {seed, offset, theta};
  sdr_dist d;
  memset(&d, 0, sizeof(d));
  d.kind = SDR_UNIFORM01;
  const size_t n = (size_t)(G0 * nc);
  float *dev = NULL, *host = (float*)malloc(n * sizeof(float));
  if (cudaMalloc((void**)&dev, n * sizeof(float)) != cudaSuccess) return 2;
  CHECK(sdr_fill(dev, SDR_F32, &d, &r, &v, NULL));
  if (cudaMemcpy(host, dev, n * sizeof(float), cudaMemcpyDeviceToHost) != cudaSuccess) return 2;
  size_t bad = 0;
  for (int64_t i = 0; i < G0; ++i)
    for (int64_t c = 0; c < nc; ++c) {
      const uint64_t j = (uint64_t)(i * G1 + c0 + c);  /* global row-major index */
      uint32_t w[4];
      CHECK(sdr_philox_block_host(seed, j % theta, j / theta + offset, w));
      const float want = (float)((double)(w[0] >> 8) * 0x1p-24);
      if (memcmp(&want, &host[i * nc + c], 4) != 0) ++bad;
    }
  /* fused dropout on the same window: y = x * keep * (1/(1-p)) */
  const double p = 0.25;
  float *x = NULL, *y = NULL, *yh = (float*)malloc(n * sizeof(float));
  if (cudaMalloc((void**)&x, n * sizeof(float)) != cudaSuccess) return 2;
  if (cudaMalloc((void**)&y, n * sizeof(float)) != cudaSuccess) return 2;
  for (size_t i = 0; i < n; ++i) host[i] = 1.0f + (float)i;
  if (cudaMemcpy(x, host, n * sizeof(float), cudaMemcpyHostToDevice) != cudaSuccess) return 2;
  CHECK(sdr_dropout(x, SDR_F32, y, SDR_F32, NULL, SDR_U8, p, &r, &v, NULL));
  if (cudaMemcpy(yh, y, n * sizeof(float), cudaMemcpyDeviceToHost) != cudaSuccess) return 2;
  const uint64_t thr = (uint64_t)ceil((1.0 - p) * 9007199254740992.0);
  const float scale = (float)(1.0 / (1.0 - p));
  for (int64_t i = 0; i < G0; ++i)
    for (int64_t c = 0; c < nc; ++c) {
      const uint64_t j = (uint64_t)(i * G1 + c0 + c);
      uint32_t w[4];
      CHECK(sdr_philox_block_host(seed, j % theta, j / theta + offset, w));
      const int keep = ((((uint64_t)w[1] << 32) | w[0]) >> 11) < thr;
      const float xv = host[i * nc + c];
      const float want = (xv * (keep ? 1.0f : 0.0f)) * scale;
      if (memcmp(&want, &yh[i * nc + c], 4) != 0) ++bad;
    }
  /* errors come back as status codes, never as exceptions or aborts */
  const int32_t e = sdr_dropout(x, SDR_F32, y, SDR_F32, NULL, SDR_U8, 1.5, &r, &v, NULL);
  printf("c_abi_fill: %zu mismatches of %zu; p=1.5 -> %s\n", bad, 2 * n, sdr_strerror(e));
  cudaFree(dev); cudaFree(x); cudaFree(y);
  free(host); free(yh);
  return (bad == 0 && e == SDR_E_PARAM) ? 0 : 1;
}
