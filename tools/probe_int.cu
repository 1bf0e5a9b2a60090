// Microbenchmark: INT32 pipe throughput on sm_100a, in Philox proportion.
// Measures (a) IMAD.WIDE.U32 alone, (b) LOP3 alone, (c) Philox4x32-10 blocks/s
// with no memory traffic (the INT roofline ceiling for the RNG path).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o probe_int probe_int.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("err %s line %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

template <int ILP>
__global__ void k_imadwide(uint32_t* out, int iters, uint32_t m) {
  uint32_t a[ILP], b[ILP];
#pragma unroll
  for (int i = 0; i < ILP; ++i) { a[i] = threadIdx.x + i; b[i] = blockIdx.x ^ i; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i) {
      uint64_t p = (uint64_t)a[i] * m;
      a[i] = (uint32_t)(p >> 32) ^ b[i];
      b[i] = (uint32_t)p;
    }
  }
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s ^= a[i] ^ b[i];
  if (s == 0x12345678u) out[0] = s;
}

__device__ __forceinline__ void philox_round(uint32_t& c0, uint32_t& c1, uint32_t& c2, uint32_t& c3, uint32_t k0, uint32_t k1) {
  uint64_t p0 = (uint64_t)c0 * 0xD2511F53u;
  uint64_t p1 = (uint64_t)c2 * 0xCD9E8D57u;
  uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1 ^ k0;
  uint32_t n2 = (uint32_t)(p0 >> 32) ^ c3 ^ k1;
  c1 = (uint32_t)p1; c3 = (uint32_t)p0; c0 = n0; c2 = n2;
}

template <int ILP>
__global__ void k_philox(uint32_t* out, int iters, uint32_t k0, uint32_t k1) {
  uint32_t acc = 0;
  uint32_t base = (blockIdx.x * blockDim.x + threadIdx.x) * ILP;
  for (int it = 0; it < iters; ++it) {
    uint32_t c0[ILP], c1[ILP], c2[ILP], c3[ILP];
#pragma unroll
    for (int i = 0; i < ILP; ++i) { c0[i] = it; c1[i] = 0; c2[i] = base + i; c3[i] = 0; }
    uint32_t kk0 = k0, kk1 = k1;
#pragma unroll
    for (int r = 0; r < 10; ++r) {
#pragma unroll
      for (int i = 0; i < ILP; ++i) philox_round(c0[i], c1[i], c2[i], c3[i], kk0, kk1);
      kk0 += 0x9E3779B9u; kk1 += 0xBB67AE85u;
    }
#pragma unroll
    for (int i = 0; i < ILP; ++i) acc ^= c0[i] + c1[i];
  }
  if (acc == 0x12345678u) out[0] = acc;
}

template <typename K>
float timeit(K launch, int reps) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  launch();
  cudaDeviceSynchronize();
  cudaEventRecord(a);
  for (int i = 0; i < reps; ++i) launch();
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  return ms / reps;
}

int main() {
  cudaDeviceProp prop; CK(cudaGetDeviceProperties(&prop, 0));
  int sms = prop.multiProcessorCount;
  int clk_khz = 0; cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  printf("device %s sms %d clock_khz %d\n", prop.name, sms, clk_khz);
  uint32_t* out; CK(cudaMalloc(&out, 64));
  const int threads = 256;
  for (int bpsm : {4, 8}) {
    int blocks = sms * bpsm;
    int iters = 4096;
    {
      float ms = timeit([&] { k_imadwide<8><<<blocks, threads>>>(out, iters, 0xD2511F53u); }, 5);
      double ops = (double)blocks * threads * iters * 8;
      printf("imadwide ilp8 bpsm %d: %.3f ms  %.1f G IMAD.WIDE/s  (%.1f per SM per clk @%d MHz)\n", bpsm, ms, ops / ms / 1e6,
             ops / (ms * 1e-3) / sms / (clk_khz * 1e3), clk_khz / 1000);
    }
    iters = 256;
    {
      float ms = timeit([&] { k_philox<4><<<blocks, threads>>>(out, iters, 1, 2); }, 5);
      double blk = (double)blocks * threads * iters * 4;
      printf("philox ilp4 bpsm %d: %.3f ms  %.1f G blocks/s = %.2f T int32-op/s (80 ops/block)\n", bpsm, ms, blk / ms / 1e6,
             blk * 80 / (ms * 1e-3) / 1e12);
    }
    {
      float ms = timeit([&] { k_philox<8><<<blocks, threads>>>(out, iters, 1, 2); }, 5);
      double blk = (double)blocks * threads * iters * 8;
      printf("philox ilp8 bpsm %d: %.3f ms  %.1f G blocks/s = %.2f T int32-op/s\n", bpsm, ms, blk / ms / 1e6,
             blk * 80 / (ms * 1e-3) / 1e12);
    }
    {
      float ms = timeit([&] { k_philox<2><<<blocks, threads>>>(out, iters, 1, 2); }, 5);
      double blk = (double)blocks * threads * iters * 2;
      printf("philox ilp2 bpsm %d: %.3f ms  %.1f G blocks/s = %.2f T int32-op/s\n", bpsm, ms, blk / ms / 1e6,
             blk * 80 / (ms * 1e-3) / 1e12);
    }
  }
  return 0;
}
