// probe.cu -- INT32 pipe microbenchmark for the roofline denominator.
//
// The RNG path is bound by the integer pipes, not HBM: one Philox4x32-10 block
// per element = 20 IMAD.WIDE.U32 (fma-heavy pipe) + 20 LOP3 (alu pipe).  These
// kernels measure both pipes with independent per-thread chains (nothing
// warp-uniform, so no work can be hoisted), plus a memory-free Philox.
#include "sdr_core.cuh"

namespace sdr {

// IMAD.WIDE throughput: ILP independent chains x <- hi(M0 x) ^ lo(M0 x) ^ it,
// one IMAD.WIDE.U32 + one LOP3 per step (the LOP3 is on the alu pipe, which
// has twice the issue rate, so the fma-heavy pipe is the limiter).  The loop
// counter enters every step, so nothing is loop-invariant.
template <int ILP>
__global__ void __launch_bounds__(256) k_probe_imad(uint32_t* sink, int iters) {
  uint32_t x[ILP];
#pragma unroll
  for (int i = 0; i < ILP; ++i) x[i] = threadIdx.x * 7u + blockIdx.x * 131u + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i) {
      const uint64_t p = mul_wide(x[i], kM0);
      x[i] = hi32(p) ^ lo32(p) ^ static_cast<uint32_t>(it);
    }
  }
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s ^= x[i];
  if (s == 0x9E3779B9u) sink[0] = s;
}

// LOP3 throughput: ILP independent 3-register chains of non-linear LUTs
// (majority 0xE8 and mux 0xCA) issued as explicit lop3.b32, so ptxas cannot
// fold iterations algebraically (an XOR-only chain is GF(2)-linear and was
// collapsed by the compiler in round 1).
__device__ __forceinline__ uint32_t lop3_maj(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm volatile("lop3.b32 %0, %1, %2, %3, 0xE8;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}
__device__ __forceinline__ uint32_t lop3_mux(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm volatile("lop3.b32 %0, %1, %2, %3, 0xCA;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}

template <int ILP>
__global__ void __launch_bounds__(256) k_probe_lop3(uint32_t* sink, int iters, uint32_t k) {
  uint32_t a[ILP], b[ILP], c[ILP];
#pragma unroll
  for (int i = 0; i < ILP; ++i) {
    a[i] = threadIdx.x * 0x9E3779B1u + i;
    b[i] = blockIdx.x * 0x85EBCA6Bu ^ (k + i);
    c[i] = ~a[i] ^ (b[i] << 3);
  }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i) {
      a[i] = lop3_maj(a[i], b[i], c[i]);
      b[i] = lop3_mux(b[i], c[i], a[i]);
      c[i] = lop3_maj(c[i], a[i], ~b[i]);  // the NOT folds into the LUT
      a[i] = lop3_mux(a[i], b[i], c[i]);
    }
  }
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s ^= a[i] ^ b[i] ^ c[i];
  if (s == 0x12345u) sink[0] = s;
}

template <int ILP>
__global__ void __launch_bounds__(256) k_probe_philox(uint32_t* sink, int iters, RoundKeys K) {
  uint32_t acc = 0;
  const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
  for (int it = 0; it < iters; ++it) {
    uint32_t x0[ILP], x1[ILP], x2[ILP], x3[ILP];
#pragma unroll
    for (int i = 0; i < ILP; ++i) {
      // every counter word per-thread varying: nothing uniform to hoist
      x0[i] = tid * 0x9E3779B1u + it;
      x1[i] = tid ^ it;
      x2[i] = tid * ILP + i;
      x3[i] = it * 0x85EBCA6Bu + tid;
    }
#pragma unroll
    for (int r = 0; r < 10; ++r) {
#pragma unroll
      for (int i = 0; i < ILP; ++i) philox_round(x0[i], x1[i], x2[i], x3[i], K.k0[r], K.k1[r]);
    }
#pragma unroll
    for (int i = 0; i < ILP; ++i) acc ^= x0[i] ^ x1[i] ^ x2[i] ^ x3[i];
  }
  if (acc == 0x12345u) sink[0] = acc;
}

template <typename F>
static float time_ms(F launch, int reps, cudaStream_t s) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  launch();
  cudaEventRecord(a, s);
  for (int i = 0; i < reps; ++i) launch();
  cudaEventRecord(b, s);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  return ms / reps;
}

int probe_int32(int device, double* imad_per_s, double* lop3_per_s, double* philox_per_s) {
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(device);
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  uint32_t* sink = nullptr;
  cudaError_t e = cudaMalloc(&sink, 64);
  if (e != cudaSuccess) {
    set_cuda_error(e);
    cudaSetDevice(prev);
    return SDR_E_CUDA;
  }
  cudaStream_t s = 0;
  const int blocks = sms * 4, threads = 256;
  const int it_mul = 4096, it_lop = 2048, it_phx = 128;
  const float t_mul = time_ms([&] { k_probe_imad<8><<<blocks, threads, 0, s>>>(sink, it_mul); }, 5, s);
  const float t_lop = time_ms([&] { k_probe_lop3<8><<<blocks, threads, 0, s>>>(sink, it_lop, 0x1234u); }, 5, s);
  const RoundKeys K = make_keys(0x243F6A8885A308D3ull);
  const float t_phx = time_ms([&] { k_probe_philox<4><<<blocks * 2, threads, 0, s>>>(sink, it_phx, K); }, 5, s);
  e = cudaGetLastError();
  cudaFree(sink);
  cudaSetDevice(prev);
  if (e != cudaSuccess) {
    set_cuda_error(e);
    return SDR_E_CUDA;
  }
  const double nthr = static_cast<double>(blocks) * threads;
  if (imad_per_s) *imad_per_s = nthr * it_mul * 8 / (t_mul * 1e-3);
  if (lop3_per_s) *lop3_per_s = nthr * it_lop * 8 * 4 / (t_lop * 1e-3);
  if (philox_per_s) *philox_per_s = 2 * nthr * it_phx * 4 / (t_phx * 1e-3);
  return SDR_OK;
}

}  // namespace sdr
