// Issue/dispatch microbenchmark for sm_100a: cycles per warp-instruction per
// SMSP for independent streams of LOP3, IMAD.WIDE, IMAD, DFMA, FFMA, IADD3 and
// their 1:1 mixes (8 independent chains per thread, 16 warps per SMSP).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench_issue tools/ubench_issue.cu
#include <cstdio>
#include <cstdint>

#define CH 8
#define ITERS 256

template <int MIX>
__global__ void __launch_bounds__(512) k(uint64_t* out, uint32_t seed) {
  uint32_t a[CH], b[CH], c[CH];
  double d[CH];
  float f[CH];
#pragma unroll
  for (int i = 0; i < CH; ++i) {
    a[i] = seed * (threadIdx.x + i + 1);
    b[i] = a[i] ^ 0x9E3779B9u;
    c[i] = a[i] + 7u;
    d[i] = (double)a[i] * 1e-9;
    f[i] = (float)a[i] * 1e-9f;
  }
  __syncthreads();
  const uint64_t t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) {
      if (MIX & 1) asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(a[i]) : "r"(b[i]), "r"(c[i]));
      if (MIX & 2) {
        uint64_t p;
        asm volatile("mul.wide.u32 %0, %1, %2;" : "=l"(p) : "r"(b[i]), "r"(0xD2511F53u));
        b[i] = (uint32_t)(p >> 32) ^ (uint32_t)p;  // (the xor is fused by ptxas? checked in SASS)
      }
      if (MIX & 4) asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(d[i]) : "d"(1.0000001), "d"(1e-12));
      if (MIX & 8) asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(f[i]) : "f"(f[(i + 1) % CH]), "f"(1e-7f));
      if (MIX & 16) asm volatile("add.u32 %0, %0, %1;" : "+r"(c[i]) : "r"(a[(i + 3) % CH]));
      if (MIX & 32) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(c[i]) : "r"(0x9E3779B9u), "r"(a[(i + 1) % CH]));
      if (MIX & 64) asm volatile("rsqrt.approx.ftz.f32 %0, %0;" : "+f"(f[i]));
      if (MIX & 128) {  // I2FP in a chain: a -> float -> bits (+LOP3 to keep it from folding)
        float t;
        asm volatile("cvt.rn.f32.u32 %0, %1;" : "=f"(t) : "r"(a[i]));
        a[i] = __float_as_uint(t) ^ b[i];
      }
      if (MIX & 256) asm volatile("shf.r.wrap.b32 %0, %0, %1, 3;" : "+r"(a[i]) : "r"(b[i]));
      if (MIX & 512) {  // F2F pair in a chain: f64 -> f32 -> f64
        float t;
        asm volatile("cvt.rn.f32.f64 %0, %1;" : "=f"(t) : "d"(d[i]));
        asm volatile("cvt.f64.f32 %0, %1;" : "=d"(d[i]) : "f"(t));
      }
      if (MIX & 2048) asm volatile("add.rm.f32 %0, %0, %1;" : "+f"(f[i]) : "f"(f[(i + 3) % CH]));
      if (MIX & 4096) asm volatile("mul.f32 %0, %0, %1;" : "+f"(f[i]) : "f"(f[(i + 5) % CH]));
      if (MIX & 8192) {  // random shared-memory LDS.64 (a 4 KiB table): bank conflicts as in the table lookups
        extern __shared__ uint2 tab[];
        const uint2 v = tab[(a[i] >> 7) & 511];
        a[i] ^= v.x;
      }
      if (MIX & 16384) asm volatile("prmt.b32 %0, %0, %1, 0x1044;" : "+r"(c[i]) : "r"(b[i]));
    }
  }
  const uint64_t t1 = clock64();
  uint32_t acc = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) acc ^= a[i] ^ b[i] ^ c[i] ^ (uint32_t)(d[i] > 2.0) ^ (uint32_t)(f[i] > 2.0f);
  if (acc == 0x12345678u) out[1] = acc;
  if (threadIdx.x == 0) atomicMax((unsigned long long*)out, (unsigned long long)(t1 - t0));
}

template <int MIX>
void run(const char* name, int per_iter_instr) {
  uint64_t* d;
  cudaMalloc(&d, 16);
  cudaMemset(d, 0, 16);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  k<MIX><<<sms, 512, 4096>>>(d, 12345u);  // warm-up
  cudaMemset(d, 0, 16);
  k<MIX><<<sms, 512, 4096>>>(d, 12345u);   // 16 warps per SM = 4 per SMSP
  uint64_t cyc;
  cudaMemcpy(&cyc, d, 8, cudaMemcpyDeviceToHost);
  // per SMSP: 4 warps x ITERS x CH x per_iter_instr warp-instructions
  const double wi = 4.0 * ITERS * CH * per_iter_instr;
  printf("%-34s %8.3f cycles per warp-instr per SMSP (%llu cycles)\n", name, cyc / wi, (unsigned long long)cyc);
  cudaFree(d);
}

int main() {
  run<1>("LOP3", 1);
  run<16>("IADD", 1);
  run<32>("IMAD (lo)", 1);
  run<2>("IMAD.WIDE (+LOP xor)", 2);
  run<4>("DFMA", 1);
  run<8>("FFMA (3 reg)", 1);
  run<1 | 16>("LOP3 + IADD", 2);
  run<1 | 32>("LOP3 + IMAD", 2);
  run<1 | 4>("LOP3 + DFMA", 2);
  run<1 | 8>("LOP3 + FFMA", 2);
  run<4 | 8>("DFMA + FFMA", 2);
  run<32 | 4>("IMAD + DFMA", 2);
  run<32 | 8>("IMAD + FFMA", 2);
  run<1 | 4 | 8>("LOP3 + DFMA + FFMA", 3);
  run<1 | 32 | 4>("LOP3 + IMAD + DFMA", 3);
  run<2 | 4>("IMAD.WIDE(+xor) + DFMA", 3);
  run<64>("MUFU.RSQ", 1);
  run<128>("I2FP + LOP3 (chain)", 2);
  run<256>("SHF (funnel)", 1);
  run<512>("F2F.F32.F64 + F2F.F64.F32 (chain)", 2);
  run<2048>("FADD.RM", 1);
  run<4096>("FMUL", 1);
  run<8192>("LDS.64 random (+LOP3)", 2);
  run<16384>("PRMT", 1);
  run<8 | 64>("FFMA + MUFU.RSQ", 2);
  return 0;
}
