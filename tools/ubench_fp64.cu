// ubench_fp64.cu -- microbenchmarks behind the Normal-transform design
// (DESIGN.md §4): FP64 issue cost with register vs constant operands, random
// shared-memory table lookups, and IMAD.WIDE next to FP64.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench_fp64 tools/ubench_fp64.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__constant__ double c_k[4] = {1.0000001, 0.9999999, 1e-300, 3.0};

template <int MODE>
__global__ void __launch_bounds__(256) k_dfma(double* sink, int iters, double a, double b) {
  double d[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) d[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if constexpr (MODE == 0) d[i] = fma(d[i], a, b);        // 3 register operands
      else if constexpr (MODE == 1) d[i] = fma(d[i], a, c_k[2]);  // constant-bank addend
      else if constexpr (MODE == 2) d[i] = d[i] * a;            // DMUL
      else d[i] = fma(d[i], d[(i + 1) & 7], b);                 // 3 distinct registers, cross-chain
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += d[i];
  if (s == 1.2345) sink[0] = s;
}

// Random 16 B lookups in a shared table of TB bytes.
template <int TB>
__global__ void __launch_bounds__(256) k_lds(double* sink, int iters) {
  extern __shared__ double2 tab[];
  for (int i = threadIdx.x; i < TB / 16; i += blockDim.x) tab[i] = make_double2(i, -i);
  __syncthreads();
  uint32_t h = threadIdx.x * 0x9E3779B9u + blockIdx.x;
  double acc = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      h = h * 1664525u + 1013904223u;
      const double2 v = tab[(h >> 8) & (TB / 16 - 1)];
      acc += v.x;
    }
  }
  if (acc == 1.2345) sink[0] = acc;
}

// IMAD.WIDE chains alone, and interleaved with DFMA chains (pipe overlap).
template <int MIX>
__global__ void __launch_bounds__(256) k_imad(double* sink, int iters, double a, double b) {
  uint32_t x[8];
  double d[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    x[i] = threadIdx.x * 7 + i;
    d[i] = i;
  }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const uint64_t p = static_cast<uint64_t>(x[i]) * 0xD2511F53u;
      x[i] = static_cast<uint32_t>(p >> 32) ^ static_cast<uint32_t>(p) ^ it;
      if constexpr (MIX) d[i] = fma(d[i], a, b);
    }
  }
  uint32_t s = 0;
  double t = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    s ^= x[i];
    t += d[i];
  }
  if (s == 12345u || t == 1.2345) sink[0] = s + t;
}

template <typename F>
static float time_ms(F launch) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  launch();
  cudaEventRecord(e0);
  for (int i = 0; i < 5; ++i) launch();
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  return ms / 5;
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* sink;
  cudaMalloc(&sink, 64);
  const int blocks = sms * 4, threads = 256, it = 4096;
  const double nthr = double(blocks) * threads;
  auto rate = [&](float ms, double ops_per_thread) { return nthr * ops_per_thread / (ms * 1e-3) / 1e12; };
  const double per_clk = 1.0 / (sms * 1.965e9) * 1e12;  // T/s -> ops per SM per clock
  float t;
  t = time_ms([&] { k_dfma<0><<<blocks, threads>>>(sink, it, 1.0000001, 1e-300); });
  printf("DFMA 3-reg       %7.3f T/s  %6.2f /SM/clk\n", rate(t, it * 8.0), rate(t, it * 8.0) * per_clk);
  t = time_ms([&] { k_dfma<1><<<blocks, threads>>>(sink, it, 1.0000001, 1e-300); });
  printf("DFMA const addend%7.3f T/s  %6.2f /SM/clk\n", rate(t, it * 8.0), rate(t, it * 8.0) * per_clk);
  t = time_ms([&] { k_dfma<2><<<blocks, threads>>>(sink, it, 1.0000001, 1e-300); });
  printf("DMUL             %7.3f T/s  %6.2f /SM/clk\n", rate(t, it * 8.0), rate(t, it * 8.0) * per_clk);
  t = time_ms([&] { k_dfma<3><<<blocks, threads>>>(sink, it, 0.5, 1e-300); });
  printf("DFMA cross-chain %7.3f T/s  %6.2f /SM/clk\n", rate(t, it * 8.0), rate(t, it * 8.0) * per_clk);
  cudaFuncSetAttribute(k_lds<65536>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  cudaFuncSetAttribute(k_lds<131072>, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072);
  t = time_ms([&] { k_lds<8192><<<blocks, threads, 8192>>>(sink, it); });
  printf("LDS.128 rnd 8K   %7.3f T/s  %6.2f /SM/clk (per-thread loads)\n", rate(t, it * 4.0), rate(t, it * 4.0) * per_clk);
  t = time_ms([&] { k_lds<65536><<<sms, 1024, 65536>>>(sink, it); });
  printf("LDS.128 rnd 64K  %7.3f T/s  %6.2f /SM/clk\n", double(sms) * 1024 * it * 4 / (t * 1e-3) / 1e12,
         double(sms) * 1024 * it * 4 / (t * 1e-3) / 1e12 * per_clk);
  t = time_ms([&] { k_lds<131072><<<sms, 1024, 131072>>>(sink, it); });
  printf("LDS.128 rnd 128K %7.3f T/s  %6.2f /SM/clk\n", double(sms) * 1024 * it * 4 / (t * 1e-3) / 1e12,
         double(sms) * 1024 * it * 4 / (t * 1e-3) / 1e12 * per_clk);
  t = time_ms([&] { k_imad<0><<<blocks, threads>>>(sink, it, 1.0000001, 1e-300); });
  printf("IMAD.WIDE        %7.3f T/s  %6.2f /SM/clk\n", rate(t, it * 8.0), rate(t, it * 8.0) * per_clk);
  t = time_ms([&] { k_imad<1><<<blocks, threads>>>(sink, it, 1.0000001, 1e-300); });
  printf("IMAD.WIDE+DFMA   %7.3f T/s  %6.2f /SM/clk (pairs)\n", rate(t, it * 8.0), rate(t, it * 8.0) * per_clk);
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
