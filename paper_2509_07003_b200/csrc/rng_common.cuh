// rng_common.cuh -- pieces shared by the fill (rng_kernels.cu) and dropout
// (dropout.cu) kernels: the chunked Philox with hoisted rounds, output dtype
// conversions, vector loads/stores, the window index map, and the host-side
// grid / launch helpers.
#pragma once

#include <cstring>

#include "sdr_core.cuh"

#ifndef SDR_PDL
// Programmatic dependent launch for the dropout and fill fast kernels.  Every
// PDL-launched kernel executes griddepcontrol.wait before touching memory the
// previous grid may use, so early launch never reorders data accesses.
#define SDR_PDL 1
#endif

namespace sdr {

// ---------------------------------------------------------------------------
// Generator parameters shared by fill and dropout.
// ---------------------------------------------------------------------------
struct Gen {
  uint64_t theta;
  uint64_t offset;
  FastDiv64 div_theta;
  RoundKeys keys;
};

inline Gen make_gen(const sdr_rng& r) {
  Gen g;
  g.theta = r.theta;
  g.offset = r.offset;
  g.div_theta = FastDiv64(r.theta);
  g.keys = make_keys(r.seed);
  return g;
}

// Rounds [R0, 10) for NE independent counters.
template <int R0, int NE>
__device__ __forceinline__ void rounds_from(const RoundKeys& K, uint32_t (&x0)[NE],
                                            uint32_t (&x1)[NE], uint32_t (&x2)[NE],
                                            uint32_t (&x3)[NE]) {
#pragma unroll
  for (int r = R0; r < 10; ++r) {
#pragma unroll
    for (int e = 0; e < NE; ++e) philox_round(x0[e], x1[e], x2[e], x3[e], K.k0[r], K.k1[r]);
  }
}

// Words 0/1 of the blocks of global indices j0 .. j0+NE-1.
template <int NE>
__device__ __forceinline__ void chunk_words(const Gen& g, uint64_t j0, uint32_t (&w0)[NE],
                                            uint32_t (&w1)[NE]) {
  uint64_t b, t;
  g.div_theta.divmod(j0, b, t);
  const uint64_t beta = b + g.offset;
  uint32_t x0[NE], x1[NE], x2[NE], x3[NE];
  const RoundKeys& K = g.keys;
  if (g.theta >= NE && t <= g.theta - NE && lo32(t) <= 0xFFFFFFFFu - (NE - 1)) {
    // Shared beta: hoist the chunk-uniform products of rounds 1 and 2.
    const uint32_t blo = lo32(beta), bhi = hi32(beta), tlo = lo32(t), thi = hi32(t);
    const uint64_t pa = mul_wide(blo, kM0);
    const uint32_t y2 = hi32(pa) ^ thi ^ K.k1[0];
    const uint32_t y3 = lo32(pa);
    const uint64_t pb0 = mul_wide(tlo, kM1);
    const uint64_t pq = mul_wide(y2, kM1);
    const uint32_t z1 = lo32(pq), hq = hi32(pq);
#pragma unroll
    for (int e = 0; e < NE; ++e) {
      const uint64_t pb = pb0 + static_cast<uint64_t>(e) * kM1;  // == M1*(tlo+e)
      const uint32_t y0 = hi32(pb) ^ bhi ^ K.k0[0];
      const uint32_t y1 = lo32(pb);
      const uint64_t pa2 = mul_wide(y0, kM0);
      x0[e] = hq ^ y1 ^ K.k0[1];
      x1[e] = z1;
      x2[e] = hi32(pa2) ^ y3 ^ K.k1[1];
      x3[e] = lo32(pa2);
    }
    rounds_from<2, NE>(K, x0, x1, x2, x3);
  } else {
#pragma unroll
    for (int e = 0; e < NE; ++e) {
      uint64_t be, te;
      g.div_theta.divmod(j0 + e, be, te);
      be += g.offset;
      x0[e] = lo32(be);
      x1[e] = hi32(be);
      x2[e] = lo32(te);
      x3[e] = hi32(te);
    }
    rounds_from<0, NE>(K, x0, x1, x2, x3);
  }
#pragma unroll
  for (int e = 0; e < NE; ++e) {
    w0[e] = x0[e];
    w1[e] = x1[e];
  }
}

// Fast path when THETA is a power of two >= NE and every chunk starts at a
// multiple of NE (host-checked): the chunk never straddles a THETA boundary,
// so beta is chunk-uniform and no 64-bit division is needed.
template <int NE>
__device__ __forceinline__ void chunk_words_aligned(const Gen& g, uint64_t j0, uint32_t (&w0)[NE],
                                                    uint32_t (&w1)[NE]) {
  const uint32_t sh = g.div_theta.s;
  const uint64_t beta = (j0 >> sh) + g.offset;
  const uint64_t t = j0 & (g.theta - 1);
  const RoundKeys& K = g.keys;
  uint32_t x0[NE], x1[NE], x2[NE], x3[NE];
  const uint32_t blo = lo32(beta), bhi = hi32(beta), tlo = lo32(t), thi = hi32(t);
  const uint64_t pa = mul_wide(blo, kM0);
  const uint32_t y2 = hi32(pa) ^ thi ^ K.k1[0];
  const uint32_t y3 = lo32(pa);
  const uint64_t pb0 = mul_wide(tlo, kM1);
  const uint64_t pq = mul_wide(y2, kM1);
  const uint32_t z1 = lo32(pq), hq = hi32(pq);
#pragma unroll
  for (int e = 0; e < NE; ++e) {
    const uint64_t pb = pb0 + static_cast<uint64_t>(e) * kM1;
    const uint32_t y0 = hi32(pb) ^ bhi ^ K.k0[0];
    const uint32_t y1 = lo32(pb);
    const uint64_t pa2 = mul_wide(y0, kM0);
    x0[e] = hq ^ y1 ^ K.k0[1];
    x1[e] = z1;
    x2[e] = hi32(pa2) ^ y3 ^ K.k1[1];
    x3[e] = lo32(pa2);
  }
  rounds_from<2, NE>(K, x0, x1, x2, x3);
#pragma unroll
  for (int e = 0; e < NE; ++e) {
    w0[e] = x0[e];
    w1[e] = x1[e];
  }
}

// chunk_words_aligned in parts: the chunk-uniform values once (hoist_chunk),
// then words of elements E0 .. E0+NE-1 (words_part), so a caller can finish
// the transform of one part before the Philox registers of the next are live.
struct ChunkHoist {
  uint32_t bhi, y3, hq, z1;
  uint64_t pb0;
};
__device__ __forceinline__ ChunkHoist hoist_chunk(const Gen& g, uint64_t j0) {
  const uint64_t beta = (j0 >> g.div_theta.s) + g.offset;
  const uint64_t t = j0 & (g.theta - 1);
  const uint64_t pa = mul_wide(lo32(beta), kM0);
  const uint32_t y2 = hi32(pa) ^ hi32(t) ^ g.keys.k1[0];
  const uint64_t pq = mul_wide(y2, kM1);
  return ChunkHoist{hi32(beta), lo32(pa), hi32(pq), lo32(pq), mul_wide(lo32(t), kM1)};
}
template <int NE, int E0>
__device__ __forceinline__ void words_part(const RoundKeys& K, const ChunkHoist& H, uint32_t (&w0)[NE],
                                           uint32_t (&w1)[NE]) {
  uint32_t x0[NE], x1[NE], x2[NE], x3[NE];
#pragma unroll
  for (int e = 0; e < NE; ++e) {
    const uint64_t pb = H.pb0 + static_cast<uint64_t>(E0 + e) * kM1;
    const uint32_t y0 = hi32(pb) ^ H.bhi ^ K.k0[0];
    const uint64_t pa2 = mul_wide(y0, kM0);
    x0[e] = H.hq ^ lo32(pb) ^ K.k0[1];
    x1[e] = H.z1;
    x2[e] = hi32(pa2) ^ H.y3 ^ K.k1[1];
    x3[e] = lo32(pa2);
  }
  rounds_from<2, NE>(K, x0, x1, x2, x3);
#pragma unroll
  for (int e = 0; e < NE; ++e) {
    w0[e] = x0[e];
    w1[e] = x1[e];
  }
}

// Word 1 only, for a keep/drop decision (dropout): the last two rounds need
// just hi(M0*x0) of round 9 and lo(M1*x2) of round 10.  Same preconditions as
// chunk_words_aligned.  A tie on the high threshold word (p = 2^-32) is
// resolved by the caller with the full block.
// Per-element part of the w1-only Philox given the chunk-uniform round-1/2
// values (bhi, y3, hq, z1) and the 64-bit M1*tau of the chunk's first element.
template <int NE>
__device__ __forceinline__ void w1_body(const RoundKeys& K, uint32_t bhi, uint32_t y3, uint32_t hq,
                                        uint32_t z1, uint64_t pb0, uint32_t (&w1)[NE]) {
  uint32_t x0[NE], x1[NE], x2[NE], x3[NE];
#pragma unroll
  for (int e = 0; e < NE; ++e) {
    const uint64_t pb = pb0 + static_cast<uint64_t>(e) * kM1;
    const uint32_t y0 = hi32(pb) ^ bhi ^ K.k0[0];
    const uint32_t y1 = lo32(pb);
    const uint64_t pa2 = mul_wide(y0, kM0);
    x0[e] = hq ^ y1 ^ K.k0[1];
    x1[e] = z1;
    x2[e] = hi32(pa2) ^ y3 ^ K.k1[1];
    x3[e] = lo32(pa2);
  }
#pragma unroll
  for (int r = 2; r < 8; ++r) {
#pragma unroll
    for (int e = 0; e < NE; ++e) philox_round(x0[e], x1[e], x2[e], x3[e], K.k0[r], K.k1[r]);
  }
#pragma unroll
  for (int e = 0; e < NE; ++e) {
    const uint32_t x2_9 = __umulhi(x0[e], kM0) ^ x3[e] ^ K.k1[8];  // round 9: x2 only
    w1[e] = x2_9 * kM1;                                              // round 10: lo(M1*x2)
  }
}

// Chunk-uniform round-1/2 values for counter (beta, tau0).
struct Hoist {
  uint32_t bhi, y3, hq, z1;
};
__device__ __forceinline__ Hoist hoist_beta(const RoundKeys& K, uint64_t beta, uint32_t thi) {
  const uint64_t pa = mul_wide(lo32(beta), kM0);
  const uint32_t y2 = hi32(pa) ^ thi ^ K.k1[0];
  const uint64_t pq = mul_wide(y2, kM1);
  return Hoist{hi32(beta), lo32(pa), hi32(pq), lo32(pq)};
}

// Word 1 only, for a keep/drop decision (dropout): the last two rounds need
// just hi(M0*x0) of round 9 and lo(M1*x2) of round 10.  Same preconditions as
// chunk_words_aligned.  A tie on the high threshold word (p = 2^-32) is
// resolved by the caller with the full block.
template <int NE>
__device__ __forceinline__ void chunk_w1_aligned(const Gen& g, uint64_t j0, uint32_t (&w1)[NE]) {
  const uint32_t sh = g.div_theta.s;
  const uint64_t beta = (j0 >> sh) + g.offset;
  const uint64_t t = j0 & (g.theta - 1);
  const Hoist H = hoist_beta(g.keys, beta, hi32(t));
  w1_body<NE>(g.keys, H.bhi, H.y3, H.hq, H.z1, mul_wide(lo32(t), kM1), w1);
}

// Words of one element at global index j (generic path).
__device__ __forceinline__ void elem_words(const Gen& g, uint64_t j, uint32_t& w0, uint32_t& w1) {
  uint64_t b, t;
  g.div_theta.divmod(j, b, t);
  b += g.offset;
  uint32_t x0 = lo32(b), x1 = hi32(b), x2 = lo32(t), x3 = hi32(t);
#pragma unroll
  for (int r = 0; r < 10; ++r) philox_round(x0, x1, x2, x3, g.keys.k0[r], g.keys.k1[r]);
  w0 = x0;
  w1 = x1;
}

// ---------------------------------------------------------------------------
// Output element types and conversions (NumPy / ml_dtypes semantics).
// ---------------------------------------------------------------------------
template <int DT> struct St;
template <> struct St<SDR_F32> { using T = float; };
template <> struct St<SDR_F64> { using T = double; };
template <> struct St<SDR_BF16> { using T = uint16_t; };
template <> struct St<SDR_F16> { using T = uint16_t; };
template <> struct St<SDR_I64> { using T = int64_t; };
template <> struct St<SDR_I32> { using T = int32_t; };
template <> struct St<SDR_U8> { using T = uint8_t; };
template <> struct St<SDR_BOOL> { using T = uint8_t; };

__device__ __forceinline__ uint16_t bf16_bits(float f) {
  return __bfloat16_as_ushort(__float2bfloat16_rn(f));
}

// float64 -> dtype with a single NumPy cast; bfloat16 goes through float32
// first exactly like ml_dtypes' float64->bfloat16 cast.
template <int DT>
__device__ __forceinline__ typename St<DT>::T from_f64(double v) {
  if constexpr (DT == SDR_F32) return __double2float_rn(v);
  else if constexpr (DT == SDR_F64) return v;
  else if constexpr (DT == SDR_BF16) return bf16_bits(__double2float_rn(v));
  else if constexpr (DT == SDR_F16) return __half_as_ushort(__double2half(v));
  else return typename St<DT>::T(0);
}

template <int DT>
__device__ __forceinline__ typename St<DT>::T one_or_zero(bool b) {
  if constexpr (DT == SDR_F32) return b ? 1.0f : 0.0f;
  else if constexpr (DT == SDR_F64) return b ? 1.0 : 0.0;
  else if constexpr (DT == SDR_BF16) return b ? uint16_t(0x3F80) : uint16_t(0);
  else if constexpr (DT == SDR_F16) return b ? uint16_t(0x3C00) : uint16_t(0);
  else return static_cast<typename St<DT>::T>(b ? 1 : 0);
}

// ---------------------------------------------------------------------------
// Vector stores of kV elements.
// ---------------------------------------------------------------------------
template <typename T, int N>
__device__ __forceinline__ void store_chunk(T* p, const T (&v)[N]) {
  constexpr int bytes = sizeof(T) * N;
  if constexpr (bytes == 4) {
    uint32_t q;
    memcpy(&q, v, 4);
    __stcs(reinterpret_cast<unsigned int*>(p), q);
  } else if constexpr (bytes == 8) {
    uint2 q;
    memcpy(&q, v, 8);
    __stcs(reinterpret_cast<uint2*>(p), q);
  } else {
    static_assert(bytes % 16 == 0, "chunk must be 4, 8 or a multiple of 16 bytes");
    uint4 q[bytes / 16];
    memcpy(q, v, bytes);
#pragma unroll
    for (int i = 0; i < bytes / 16; ++i) __stcs(reinterpret_cast<uint4*>(p) + i, q[i]);
  }
}

template <typename T, int N>
__device__ __forceinline__ void load_chunk(const T* p, T (&v)[N]) {
  constexpr int bytes = sizeof(T) * N;
  if constexpr (bytes == 4) {
    const uint32_t q = __ldcs(reinterpret_cast<const unsigned int*>(p));
    memcpy(v, &q, 4);
  } else if constexpr (bytes == 8) {
    const uint2 q = __ldcs(reinterpret_cast<const uint2*>(p));
    memcpy(v, &q, 8);
  } else {
    static_assert(bytes % 16 == 0, "chunk must be 4, 8 or a multiple of 16 bytes");
    uint4 q[bytes / 16];
#pragma unroll
    for (int i = 0; i < bytes / 16; ++i) q[i] = __ldcs(reinterpret_cast<const uint4*>(p) + i);
    memcpy(v, q, bytes);
  }
}

// Global flat index of chunk q (CH elements inside one row of the canonical
// view, nd >= 1): row/column by the launch-constant chunks-per-row divisor, the
// inner outer-dims by their sizes; the outermost digit needs no division (the
// row index is below its extent).
__device__ __forceinline__ uint64_t outer_base(const ViewIndexer& ix, const FastDiv64& div_cpr,
                                               uint64_t q, int CH) {
  uint64_t row, cq;
  div_cpr.divmod(q, row, cq);
  const CanonView& cv = ix.cv;
  uint64_t j = static_cast<uint64_t>(cv.base) + cq * CH;
  for (int k = cv.nd - 1; k >= 1; --k) {
    uint64_t qq, r;
    ix.div_o[k].divmod(row, qq, r);
    j += r * static_cast<uint64_t>(cv.ostride[k]);
    row = qq;
  }
  return j + row * static_cast<uint64_t>(cv.ostride[0]);
}

// ---------------------------------------------------------------------------
// Host helpers shared by the fill and dropout launchers.
// ---------------------------------------------------------------------------
inline int device_sms() {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms > 0 ? sms : 148;
}

// Persistent grid: one wave of resident CTAs (SMs x occupancy), or fewer
// blocks when the work is small.  Grid-stride loops cover the rest.
template <typename K>
inline int grid_for(K kernel, uint64_t work, int threads, size_t dyn_smem = 0) {
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, dyn_smem) != cudaSuccess ||
      per_sm < 1)
    per_sm = 1;
  const uint64_t cap = static_cast<uint64_t>(device_sms()) * per_sm;
  const uint64_t blocks = (work + threads - 1) / threads;
  return static_cast<int>(blocks < cap ? (blocks > 0 ? blocks : 1) : cap);
}

inline int launch_grid(uint64_t work, int threads) {
  const uint64_t blocks = (work + threads - 1) / threads;
  const uint64_t cap = static_cast<uint64_t>(device_sms()) * 8;
  return static_cast<int>(blocks < cap ? (blocks > 0 ? blocks : 1) : cap);
}

// Every chunk start j0 = base + sum(digit*ostride) + c*ch is a multiple of ch
// and THETA is a power of two >= ch: no chunk straddles a THETA boundary.
inline bool chunks_aligned(const CanonView& cv, uint64_t theta, int ch) {
  if ((theta & (theta - 1)) != 0 || theta < static_cast<uint64_t>(ch)) return false;
  if (cv.base % ch != 0) return false;
  for (int k = 0; k < cv.nd; ++k)
    if (cv.ostride[k] % ch != 0) return false;
  return true;
}

inline void setup_chunks(const CanonView& cv, bool fast, uint64_t& nchunks, uint64_t& cpr,
                         FastDiv64& div_cpr, int ch = kV) {
  if (fast) {
    cpr = static_cast<uint64_t>(cv.inner) / ch;
    nchunks = static_cast<uint64_t>(cv.numel) / ch;
  } else {
    cpr = 1;
    nchunks = 0;
  }
  div_cpr = FastDiv64(cpr > 0 ? cpr : 1);
}

// 256-thread launch with programmatic stream serialization (PDL) when SDR_PDL.
template <typename K, typename Args>
inline void launch_pdl(K kernel, int grid, cudaStream_t s, const Args& A, size_t dyn_smem = 0,
                       int threads = 256) {
#if SDR_PDL
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(grid));
  cfg.blockDim = dim3(static_cast<unsigned>(threads));
  cfg.dynamicSmemBytes = dyn_smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kernel, A);
#else
  kernel<<<grid, threads, dyn_smem, s>>>(A);
#endif
}

inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

}  // namespace sdr
