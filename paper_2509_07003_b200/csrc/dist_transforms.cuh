// dist_transforms.cuh -- device side of the distribution transforms
// (rng.py:104-182): the parameters of a fill (DistP), the certified Normal fast
// paths (float64 and the float32 path of bfloat16 outputs) with their tables
// and the exact NumPy-table fallback, the TMA staging of those tables, and
// dist_value for every (distribution, dtype).  Host-side table construction
// and calibration live in rng_kernels.cu.
#pragma once

#include "rng_common.cuh"

namespace sdr {

// ---------------------------------------------------------------------------
// Distribution parameters and the Normal mirror state.
// ---------------------------------------------------------------------------
// Device lookup tables of the Normal fast path (40 KiB, staged in shared
// memory by every kernel that draws normals).  With n = 2^24 - k the fast path
// evaluates X = 2L = -2 ln(n 2^-24) as
//   X = (-e) 2ln2 + 2 ln(inv_j) + g(s),  s = -2t = 2 - 2 m' inv_j  (exact),
//   g(s) = -2 log1p(-s/2) = s + s^2/4 + s^3/12 + s^4/32 + s^5/80,
// with n = 2^(e+24) m', m' in [0.75, 1.5) and j the top 9 fraction bits of n;
// r = sqrt(X) is one Newton step on the MUFU.RSQ64H seed.  The cosine is
//   c = cos(i pi/1024 + K d) = C_i (1 + cm(d)) - S_i sd(d),
// i = round(k / 8192), d = k - 8192 i in [-4096, 4096), K = 2 pi / 2^24.
//   logt[j] = (-2 mult_j 2^-23, 2 ln(inv_j))  (+2^-1000 at j = 0: X > 0 at k = 0)
//   trig[i] = (cos, sin)(i pi/1024), i = 0..2047 (k near 2^24 wraps to i = 0)
// Both are approximations to ~2^-45 whose exact error against the host's NumPy
// is measured over all 2^24 inputs at load time (k_normal_calibrate).
struct NormalLut {
  double2 logt[512];
  double2 trig[2048];
};

// float32 tables of the bfloat16 fast path, staged in (dynamic) shared memory:
// the log table plus a two-level cosine table, cos(2 pi k / 2^24) =
// C_hi C_lo - S_hi S_lo with k = 4096 hi + lo (68 KiB).
struct NormalLut32 {
  float2 logt[512];
  float2 trig_hi[4096];  // (cos, sin)(2 pi hi / 4096)
  float2 trig_lo[4096];  // (cos, sin)(2 pi lo / 2^24)
};

struct NormalMirror {
  const double* rtab;   // NumPy r[k] = sqrt(-2*log1p(-k*2^-24))
  const double* ctab;   // NumPy c[k] = cos(2*pi*(k*2^-24))
  const NormalLut* lut; // device copy of the fast-path tables
  const NormalLut32* lut32;
  double nh, th;        // -0.5*std, 1.5*std: the Newton step of r_fast returns std*r
  double kr, k0;        // certification bound B = (std r) kr + k0
  // float32 fast path (bfloat16 outputs): calibrated errors and bound terms
  double err_r32, err_c32;
  float mean32, std32, b32_r, b32_c;  // B32 = r*b32_r + b32_c
  unsigned long long* fallbacks;
};

struct DistP {
  int32_t kind;
  float lo32, span32;          // Uniform f32 path
  double lo, span;             // Uniform f64 path
  double mean, stdv;           // Normal
  uint64_t keep_thr;           // Bernoulli: keep <=> u64 < keep_thr (or always)
  uint32_t keep_all;
  int64_t ilo;                 // RandInt
  FastDiv64 ispan;
  NormalMirror nm;
};

constexpr double kTwo52m1 = 4503599627370495.0;     // 2^52 - 1
constexpr double kTwo52p1047 = 4503599627371543.0;  // 2^52 + 1047
constexpr double kTwo52p4096 = 4503599627374592.0;  // 2^52 + 4096
constexpr double kK1 = 0x1.921fb54442d18p-22;       // 2 pi / 2^24

// Polynomial coefficients as constant-bank operands (no per-use materialisation).
__constant__ double c_npoly[9] = {
    1.0 / 80.0, 1.0 / 32.0, 1.0 / 12.0, 0.25,        // g(s) Horner
    kK1 * kK1 * kK1 * kK1 / 24.0, -0.5 * kK1 * kK1,   // cos(K d) - 1 = d^2 (c4 d^2 + c2)
    -kK1 * kK1 * kK1 / 6.0, kK1,                      // sin(K d) = d (s3 d^2 + K)
    0x1.62e42fefa39efp0};                             // 2 ln 2
#ifndef SDR_NORMAL_BF16_F32
#define SDR_NORMAL_BF16_F32 1  // certified float32 Box-Muller for bfloat16 outputs
#endif
#ifndef SDR_NORMAL_SPLIT
#define SDR_NORMAL_SPLIT 1  // float64 phases of a chunk in SPLIT passes (register pressure)
#endif
#ifndef SDR_R_NEWTON2
#define SDR_R_NEWTON2 0   // second Newton step for r (fewer certification fallbacks)
#endif
#ifndef SDR_R32_NEWTON
#define SDR_R32_NEWTON 0  // Newton step on the float32 rsqrt seed (fewer float64 fallbacks)
#endif
#ifndef SDR_COUNT_F32_MISS
#define SDR_COUNT_F32_MISS 0  // A/B diagnostics: count float32-path misses as fallbacks
#endif
#ifndef SDR_FILL_MINB
#define SDR_FILL_MINB 2   // CTAs/SM the register budget of the fill kernels is sized for
#endif

__host__ __device__ __forceinline__ double hilo(uint32_t hi, uint32_t lo) {
#ifdef __CUDA_ARCH__
  return __hiloint2double(static_cast<int>(hi), static_cast<int>(lo));
#else
  const uint64_t b = (static_cast<uint64_t>(hi) << 32) | lo;
  double d;
  memcpy(&d, &b, 8);
  return d;
#endif
}
__host__ __device__ __forceinline__ uint32_t dhi(double d) {
#ifdef __CUDA_ARCH__
  return static_cast<uint32_t>(__double2hiint(d));
#else
  uint64_t b;
  memcpy(&b, &d, 8);
  return static_cast<uint32_t>(b >> 32);
#endif
}
__host__ __device__ __forceinline__ uint32_t dlo(double d) {
#ifdef __CUDA_ARCH__
  return static_cast<uint32_t>(__double2loint(d));
#else
  uint64_t b;
  memcpy(&b, &d, 8);
  return static_cast<uint32_t>(b);
#endif
}

__device__ __forceinline__ double rsqrt_seed(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  return y;
}

template <typename T>
__device__ __forceinline__ const T& lut_at(const T* base, uint32_t byte_off) {
  return *reinterpret_cast<const T*>(reinterpret_cast<const char*>(base) + byte_off);
}

// std * r(k), r(k) = sqrt(-2*log1p(-k*2^-24)), k = w0 >> 8, as described at
// NormalLut; nh = -0.5*std, th = 1.5*std fold std into the Newton step.  No
// select for k = 0: the 2^-1000 in logt[0] keeps X > 0 and r ~ 2^-499.5.
__device__ __forceinline__ double r_fast(uint32_t w0, const NormalLut* L, double nh, double th) {
  const double* C = c_npoly;
  const double nd = hilo(0x43300000u, (w0 >> 8) ^ 0xFFFFFFu) - kTwo52m1;  // n, exact
  const uint32_t hw = dhi(nd), lw = dlo(nd);
  const double2 tb = lut_at(L->logt, (hw >> 7) & 0x1FF0u);               // j = hw[19:11]
  const double s = fma(hilo((hw & 0x000FFFFFu) | 0x41600000u, lw), tb.x, 2.0);  // -2t, exact
  double p = fma(s, C[0], C[1]);
  p = fma(s, p, C[2]);
  p = fma(s, p, C[3]);
  const double g = fma(s * s, p, s);                                     // -2 log1p(t)
  const double ne = kTwo52p1047 - hilo(0x43300000u, (hw + 0x80000u) >> 20);  // -e, exact
  const double X = fma(ne, C[8], tb.y + g);                              // -2 ln w
  double h = rsqrt_seed(X);
#if SDR_R_NEWTON2
  h = h * fma(X * h, h * -0.5, 1.5);                                     // seed to ~2^-40
#endif
  const double gx = X * h;
  return gx * fma(gx * h, nh, th);                                       // std * sqrt(X)
}

// cos(2*pi*k*2^-24), k = w1 >> 8: nearest pi/1024 table point + residual.
__device__ __forceinline__ double c_fast(uint32_t w1, const NormalLut* L) {
  const double* C = c_npoly;
  const uint32_t u = w1 + 0x100000u;                                     // (k + 4096) << 8
  const double2 cs = lut_at(L->trig, (u >> 17) & 0x7FF0u);               // i = u >> 21
  const double d = hilo(0x43300000u, (u >> 8) & 0x1FFFu) - kTwo52p4096;  // k - 8192 i, exact
  const double d2 = d * d;
  const double cm = d2 * fma(d2, C[4], C[5]);                            // cos(K d) - 1
  const double sd = d * fma(d2, C[6], C[7]);                             // sin(K d)
  return fma(-cs.y, sd, fma(cs.x, cm, cs.x));
}

// float32 fast functions for the bfloat16 path: the same reductions as
// r_fast / c_fast in float32 arithmetic (~2^-21), calibrated exhaustively like
// the float64 ones.  Tables (NormalLut32): logt[j] = (-2 mult_j 2^-23,
// 2 ln(inv_j)) (+2^-100 at j = 0), trig[i] = (cos, sin)(i pi/1024).
__device__ __forceinline__ float r32_fast(uint32_t w0, const NormalLut32* L) {
  const uint32_t hw = __float_as_uint(__uint2float_rn(0x1000000u - (w0 >> 8)));  // n, exact
  const float2 tb = lut_at(L->logt, (hw >> 11) & 0xFF8u);                         // j = hw[22:14]
  const float s = fmaf(__uint_as_float((hw & 0x007FFFFFu) | 0x4B000000u), tb.x, 2.0f);  // -2t
  const float g = fmaf(s * s, fmaf(s, 1.0f / 12.0f, 0.25f), s);                   // -2 log1p(t)
  const float e = __uint_as_float(0x4B000000u | ((hw + 0x400000u) >> 23)) - 8388759.0f;  // e, exact
  const float X = fmaf(e, -1.38629436f, tb.y + g);                                // -2 ln w
  float h;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(h) : "f"(X));
#if SDR_R32_NEWTON
  const float gx = X * h;
  return gx * fmaf(gx * h, -0.5f, 1.5f);
#else
  return X * h;
#endif
}

__device__ __forceinline__ float c32_fast(uint32_t w1, const NormalLut32* L) {
  const float2 a = lut_at(L->trig_hi, (w1 >> 17) & 0x7FF8u);  // hi = k >> 12
  const float2 b = lut_at(L->trig_lo, (w1 >> 5) & 0x7FF8u);   // lo = k & 4095
  return fmaf(a.x, b.x, -a.y * b.y);
}

template <int DT>
__device__ __forceinline__ typename St<DT>::T normal_value(const DistP& P, const NormalLut* L,
                                                           uint32_t w0, uint32_t w1);

template <int NE>
__device__ __forceinline__ void normal_chunk_bf16(const DistP& P, const NormalLut32* L32,
                                                  const uint32_t* w0, const uint32_t* w1, uint16_t* out) {
  uint32_t badmask = 0;
#pragma unroll
  for (int e = 0; e < NE; ++e) {
    const float r = r32_fast(w0[e], L32), c = c32_fast(w1[e], L32);
    const float v = fmaf(P.nm.std32, r * c, P.nm.mean32);
    // |v - v_numpy| <= r*b32_r + b32_c   (host: bound terms)
    const float B = fmaf(r, P.nm.b32_r, P.nm.b32_c);  // |v| term folded (host)
    // bf16(RN32(.)) is monotone: [v-B, v+B] rounds to one bfloat16 iff both ends do
    const __nv_bfloat162 pk = __floats2bfloat162_rn(__fsub_rd(v, B), __fadd_ru(v, B));
    uint32_t lh;
    memcpy(&lh, &pk, 4);
    out[e] = static_cast<uint16_t>(lh);
    badmask |= ((lh ^ (lh >> 16)) & 0xFFFFu) ? (1u << e) : 0u;
  }
  if (__builtin_expect(badmask != 0, 0)) {
#if SDR_COUNT_F32_MISS
    atomicAdd(P.nm.fallbacks, static_cast<unsigned long long>(__popc(badmask)));
#endif
    // float64 certified path (tables read through L1/L2), then the exact NumPy tables
#pragma unroll
    for (int e = 0; e < NE; ++e)
      if (badmask & (1u << e)) out[e] = normal_value<SDR_BF16>(P, P.nm.lut, w0[e], w1[e]);
  }
}

// Exact Normal (rng.py:150-156) from the NumPy tables: float64 Box-Muller with
// the reference's own r[k1], c[k2], then one cast.
template <int DT>
__device__ __forceinline__ typename St<DT>::T normal_exact(const DistP& P, uint32_t w0, uint32_t w1) {
  const double r = __ldg(P.nm.rtab + (w0 >> 8)), c = __ldg(P.nm.ctab + (w1 >> 8));
  return from_f64<DT>(__dadd_rn(P.mean, __dmul_rn(P.stdv, __dmul_rn(r, c))));
}

// Certified fast value: v = fma(std r, c, mean) and |v_numpy - v| <= B; if the
// monotone cast R to DT gives R(v - B) == R(v + B) that is the reference's
// value, else ok = false.
template <int DT>
__device__ __forceinline__ typename St<DT>::T normal_certified(const DistP& P, double rs, double c,
                                                               bool& ok) {
  const double v = fma(rs, c, P.mean);
  const double B = fma(rs, P.nm.kr, P.nm.k0);  // |v| 2^-51 folded: |v| <= |mean| + rs (host)
  const auto lo = from_f64<DT>(v - B), hi = from_f64<DT>(v + B);
  if constexpr (DT == SDR_F32) ok = __float_as_uint(lo) == __float_as_uint(hi);
  else ok = lo == hi;
  return lo;
}

// Normal (rng.py:150-156): float64 Box-Muller then one cast.  Fast path with
// the table functions + a rigorous error bound; elements whose rounding to DT
// the bound cannot certify recompute from the exact NumPy tables.
template <int DT>
__device__ __forceinline__ typename St<DT>::T normal_value(const DistP& P, const NormalLut* L,
                                                           uint32_t w0, uint32_t w1) {
  if constexpr (DT != SDR_F64) {
    bool ok;
    const auto v = normal_certified<DT>(P, r_fast(w0, L, P.nm.nh, P.nm.th), c_fast(w1, L), ok);
    if (__builtin_expect(ok, 1)) return v;
    atomicAdd(P.nm.fallbacks, 1ull);
  }
  return normal_exact<DT>(P, w0, w1);
}

// A whole chunk of normals, phase by phase (all r, all c, then combine and
// certify) so the independent float64 chains interleave; one branch for the
// rare uncertified elements.
template <int DT, int NE>
__device__ __forceinline__ void normal_chunk(const DistP& P, const NormalLut* L, const uint32_t* w0,
                                             const uint32_t* w1, typename St<DT>::T* out) {
  double rs[NE], c[NE];
#pragma unroll
  for (int e = 0; e < NE; ++e) rs[e] = r_fast(w0[e], L, P.nm.nh, P.nm.th);
#pragma unroll
  for (int e = 0; e < NE; ++e) c[e] = c_fast(w1[e], L);
  uint32_t badmask = 0;
#pragma unroll
  for (int e = 0; e < NE; ++e) {
    bool ok;
    out[e] = normal_certified<DT>(P, rs[e], c[e], ok);
    badmask |= ok ? 0u : (1u << e);
  }
  if (__builtin_expect(badmask != 0, 0)) {
#pragma unroll
    for (int e = 0; e < NE; ++e) {
      if (badmask & (1u << e)) {
        atomicAdd(P.nm.fallbacks, 1ull);
        out[e] = normal_exact<DT>(P, w0[e], w1[e]);
      }
    }
  }
}
// Stage the Normal tables in shared memory: one elected thread issues a TMA
// bulk copy (cp.async.bulk global -> shared, completion on an mbarrier) and the
// CTA waits on the barrier -- one 20-40 KiB transfer instead of a loop of
// dependent per-thread loads.  Whole CTA participates.
__device__ __forceinline__ void mbar_wait_parity0(uint32_t bar) {
  uint32_t done;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done) : "r"(bar) : "memory");
  } while (!done);
}

// Issue the bulk copy (thread 0) and make the barrier visible to the CTA;
// returns the barrier to pass to stage_lut_wait.  Work that does not read the
// tables (e.g. the first chunk's Philox) can run between the two.
template <typename LUT>
__device__ __forceinline__ uint32_t stage_lut_begin(LUT* dst, const LUT* src) {
  static_assert(sizeof(LUT) % 16 == 0 && sizeof(LUT) < (1u << 20), "LUT size");
  __shared__ __align__(8) uint64_t s_bar;
  const uint32_t bar = static_cast<uint32_t>(__cvta_generic_to_shared(&s_bar));
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(bar) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
                 :: "r"(bar), "r"(static_cast<uint32_t>(sizeof(LUT))) : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
        :: "r"(static_cast<uint32_t>(__cvta_generic_to_shared(dst))), "l"(src),
           "r"(static_cast<uint32_t>(sizeof(LUT))), "r"(bar) : "memory");
  }
  __syncthreads();  // barrier initialised before anyone polls it
  return bar;
}

__device__ __forceinline__ void stage_lut_wait(uint32_t bar) { mbar_wait_parity0(bar); }

template <typename LUT>
__device__ __forceinline__ void stage_lut(LUT* dst, const LUT* src) {
  stage_lut_wait(stage_lut_begin(dst, src));
}

template <int DIST, int DT>
__device__ __forceinline__ typename St<DT>::T dist_value(const DistP& P, const NormalLut* L,
                                                         uint32_t w0, uint32_t w1) {
  using T = typename St<DT>::T;
  const uint64_t u64 = (static_cast<uint64_t>(w1) << 32) | w0;
  if constexpr (DIST == SDR_UNIFORM01) {
    if constexpr (DT == SDR_F32) {
      return __fmul_rn(__uint2float_rn(w0 >> 8), 0x1p-24f);
    } else {
      return static_cast<T>(__ull2double_rn(u64 >> 11) * 0x1p-53);
    }
  } else if constexpr (DIST == SDR_UNIFORM) {
    if constexpr (DT == SDR_F32) {
      const float u = __fmul_rn(__uint2float_rn(w0 >> 8), 0x1p-24f);
      return __fadd_rn(P.lo32, __fmul_rn(P.span32, u));
    } else {
      const double u = __ull2double_rn(u64 >> 11) * 0x1p-53;
      return from_f64<DT>(__dadd_rn(P.lo, __dmul_rn(P.span, u)));
    }
  } else if constexpr (DIST == SDR_NORMAL) {
    return normal_value<DT>(P, L, w0, w1);
  } else if constexpr (DIST == SDR_RANDINT) {
    uint64_t q, rem;
    P.ispan.divmod(u64, q, rem);
    const int64_t x = static_cast<int64_t>(static_cast<uint64_t>(P.ilo) + rem);
    if constexpr (DT == SDR_I64) return x;
    else if constexpr (DT == SDR_I32) return static_cast<int32_t>(x);
    else if constexpr (DT == SDR_F64) return __ll2double_rn(x);
    else if constexpr (DT == SDR_F32) return __ll2float_rn(x);
    else return T(0);
  } else {  // SDR_BERNOULLI
    return one_or_zero<DT>(P.keep_all || u64 < P.keep_thr);
  }
}

}  // namespace sdr
