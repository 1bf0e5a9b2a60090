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

// Tables of the float64-precision fast path of float32 / float16 outputs
// (160 KiB, staged in dynamic shared memory by 512-thread CTAs, one per SM).
// With n = 2^24 - k, nf = float(n) = 2^E m (exact, m in [1, 2)), j = the top
// 11 fraction bits of m:
//   X = -2 ln(n 2^-24) = (24 - E) 2ln2 + T_j - 2 log1p(s),  s = m inv_j - 1,
// inv_j ~ 1/m_j a multiple of 2^-12 (so s is an exact float32 FFMA, |s| <
// 2^-11), T_j = 2 ln(inv_j) in float64.  Buckets with m >= 1.5 use inv_j ~
// 1/m_j in (1/2, 2/3] and T_j = 2 ln(2 inv_j) - C2 (C2 = RN(2 ln 2), the
// constant the (24 - E) term is multiplied by), so the top bucket (inv = 1/2,
// T = -C2, E = 23) gives A = 0 exactly and X near 0 keeps full relative
// precision.  The cosine is two-level: cos(2 pi k2 / 2^24) = C_i C_b - S_i S_b
// with k2 = 4096 i + b.
struct __align__(16) LogEnt2 {
  float inv;
  float pad;
  double T;
};
struct NormalLut2 {
  LogEnt2 logt[2048];
#if SDR_N2_COS2
  double2 cos_hi[4096];  // (cos, sin)(2 pi i / 4096)
  double2 cos_lo[4096];  // (cos, sin)(2 pi b / 2^24)
#else
  double2 trig[2048];    // (cos, sin)(i pi/1024), as NormalLut::trig (c_fast)
#endif
};

// The exact mirror of NumPy's two transcendentals (rng.py:154-155) in 2-bit
// ulp corrections against the device's own libm: for k in [0, 2^24)
//   L(k) = log1p(-k 2^-24),  C(k) = cos((2 pi) (k 2^-24)),
// code = bits(NumPy) - bits(CUDA) in {0, +1, -1}, 3 = exception (exact value
// in a sorted (key, value) list).  8 MiB per device instead of 2 x 128 MiB of
// float64 tables; r = sqrt(-2 L) is correctly rounded on both sides.
struct ExactMirror {
  const uint32_t* code_l;  // 16 codes per word
  const uint32_t* code_c;
  const uint32_t* xk_l;    // exceptions: sorted keys, values
  const double* xv_l;
  const uint32_t* xk_c;
  const double* xv_c;
  int32_t nx_l, nx_c;
};

// Per-point float64 corrections of r (normal_chunk_f64): 8 bits against
// r_unit's two Newton steps (SDR_F64_R8), else 16 bits against one.
#ifndef SDR_F64_R8
#define SDR_F64_R8 1
#endif
#if SDR_F64_R8
using DeltaR = int8_t;
#else
using DeltaR = int16_t;
#endif
constexpr int kDeltaEscR = SDR_F64_R8 ? -128 : -32768;
constexpr int kDeltaMaxR = SDR_F64_R8 ? 127 : 32767;

// float64 outputs, cosine: c_cr evaluates cos(RN(2pi u2)) -- NumPy's own
// argument -- in double-double from a (cos, sin)(i pi/1024) table stored as
// double-doubles (absolute error < 2^-76).  Rounded to nearest it equals
// NumPy's (glibc's) value except within a narrow band around rounding
// midpoints (glibc misses there) and where |c| < 2^-10 (the table's precision
// runs out); those elements are flagged and read a correction instead.  The
// load verifies on all 2^24 points that every unflagged one matches.
struct __align__(16) CosDD {
  double ch, cl, sh, sl;
};
constexpr int kCosDD = 2049;
// pi/1024 = kQ1 + kQ2 + kQ3 (40 + 40 + 29 significant bits, from quad precision)
constexpr double kQ1 = 0x1.921fb54442p-9, kQ2 = 0x1.a308d31318p-50, kQ3 = 0x1.8a2e037p-90;
#ifndef SDR_COS_TAU
#define SDR_COS_TAU 0.03  // c_cr's flag band around rounding midpoints, in ulps (glibc misses within 0.016)
#endif

struct NormalMirror {
  const double* rtab;   // full NumPy r[k] table, only when the compact mirror failed verification
  const double* ctab;   // full NumPy c[k] table (same)
  ExactMirror em;
  const NormalLut* lut; // device copy of the fast-path tables
  const NormalLut32* lut32;
  const NormalLut2* lut2;
  double kr2, k02;      // certification bound of the NormalLut2 path
  double nh, th;        // -0.5*std, 1.5*std: the Newton step of r_fast returns std*r
  double kr, k0;        // certification bound B = (std r) kr + k0
  // float32 fast path (bfloat16 outputs): calibrated errors and bound terms
  double err_r32, err_c32;
  float mean32, std32, b32_r, b32_c;  // B32 = r*b32_r + b32_c
  float bm_r, bm_c, bm_i;             // r32_mufu path: B = r bm_r + h bm_i + bm_c
  float bmc_r, bmc_i;                 // the same with the MUFU cosine (SDR_BF16_COS_MUFU)
  const DeltaR* dr;                   // float64 outputs: per-point corrections (normal_chunk_f64), or null
  const int16_t* dc;                  // against c_fast (no c_cr)
  const CosDD* cdd;                   // c_cr's table when it verified at load (its 8-bit corrections
                                      // follow dr: dc8()), else null
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
#ifndef SDR_BF16_COS_MUFU
#define SDR_BF16_COS_MUFU 1  // bfloat16 normals: cosine from MUFU cos.approx (else the two-level table)
#endif
#ifndef SDR_NORMAL_BF16_MUFU
#define SDR_NORMAL_BF16_MUFU 1  // bfloat16 normals: r from MUFU lg2 / rsqrt (r32_mufu) instead of the log table
#endif
#ifndef SDR_C32_POLY
#define SDR_C32_POLY 0   // c32_fast: low part of the angle by polynomial (A/B: 1-3% slower than the second table)
#endif
#ifndef SDR_MISSQ
#define SDR_MISSQ 1      // bfloat16 fast fills: queue uncertified elements per warp, resolve 32 at a time
#endif
#ifndef SDR_NORMAL_SPLIT
#define SDR_NORMAL_SPLIT 1  // float64 phases of a chunk in SPLIT passes (register pressure)
#endif
#ifndef SDR_R_SEED32
#define SDR_R_SEED32 1    // r_fast: float32 rsqrt seed (1) or MUFU.RSQ64H (0)
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
#ifndef SDR_F64N_MINB
#define SDR_F64N_MINB 2   // CTAs/SM for the float64 Normal fills (latency-bound on their L2 gathers)
#endif
#ifndef SDR_NORMAL_N2
#define SDR_NORMAL_N2 0   // float32/float16 normals on the NormalLut2 tables (else NormalLut)
#endif
#ifndef SDR_FILL_PIPE
#define SDR_FILL_PIPE 0   // software-pipelined Normal walk loop (next chunk's Philox beside this transform)
#endif
#ifndef SDR_NSPLIT
#define SDR_NSPLIT 1      // Normal chunks in NSPLIT parts (Philox + transform per part: fewer live registers)
#endif
#ifndef SDR_BF16_MINB
#define SDR_BF16_MINB 3  // CTAs/SM for the bfloat16 Normal kernels' register budget (no tables to stage)
#endif
#ifndef SDR_N2_MINB
#define SDR_N2_MINB 2     // CTAs/SM the NormalLut2 kernels' register budget is sized for (256 threads)
#endif
#ifndef SDR_R2_SEED
#define SDR_R2_SEED 1     // r_fast2 rsqrt seed: 0 MUFU.RSQ64H, 1 float32 MUFU.RSQ, 2 RSQ64H + 2nd Newton
#endif
#ifndef SDR_N2_COS2
#define SDR_N2_COS2 0     // NormalLut2 cosine: two-level table (1) or c_fast's table + polynomial (0)
#endif
#ifndef SDR_N2_THREADS
#define SDR_N2_THREADS 256  // CTA size of the NormalLut2 kernels (smem allows 2-3 CTAs/SM without COS2)
#endif

// Kernels drawing float32 / float16 normals stage NormalLut2 (64 KiB; 160 KiB
// with SDR_N2_COS2, then one 512-thread CTA per SM).  Everything else:
// 256-thread CTAs, SDR_FILL_MINB per SM.
// 16-bit outputs whose Normal fast path runs in float32 (the bfloat16 path;
// float16 too with SDR_NORMAL_F16_F32)
#ifndef SDR_NORMAL_F16_F32
#define SDR_NORMAL_F16_F32 1
#endif
template <int DT>
constexpr bool half_dt() {
  return DT == SDR_BF16 || (SDR_NORMAL_F16_F32 && DT == SDR_F16);
}
// MUFU cosine on the float32 path (float16 may use the table cosine: its
// narrower misses band, SDR_F16_COS_MUFU=0)
#ifndef SDR_F16_COS_MUFU
#define SDR_F16_COS_MUFU 1
#endif
template <int DT>
constexpr bool cos_mufu() {
  return SDR_BF16_COS_MUFU && (DT == SDR_BF16 || SDR_F16_COS_MUFU);
}
template <int DIST, int DT>
constexpr bool uses_lut2() {
  return SDR_NORMAL_N2 && DIST == SDR_NORMAL && (DT == SDR_F32 || (DT == SDR_F16 && !half_dt<DT>()));
}
// bfloat16 normals with both functions from MUFU need no tables in shared
// memory (the rare float64 fallbacks read theirs through L1).
template <int DIST, int DT>
constexpr bool tablefree() {
  return SDR_NORMAL_BF16_MUFU && cos_mufu<DT>() && SDR_NORMAL_BF16_F32 && DIST == SDR_NORMAL && half_dt<DT>();
}
template <int DIST, int DT>
constexpr bool stages_lut() { return DIST == SDR_NORMAL && !tablefree<DIST, DT>(); }
template <int DIST, int DT>
constexpr int fill_threads() { return uses_lut2<DIST, DT>() ? SDR_N2_THREADS : 256; }
template <int DIST, int DT>
constexpr int fill_minb() {
  return uses_lut2<DIST, DT>() ? SDR_N2_MINB * 256 / SDR_N2_THREADS
         : (DIST == SDR_NORMAL && half_dt<DT>() && SDR_NORMAL_BF16_F32) ? SDR_BF16_MINB
         : (DIST == SDR_NORMAL && DT == SDR_F64) ? SDR_F64N_MINB : SDR_FILL_MINB;
}

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

// MUFU.RSQ without the denormal fix-up rsqrtf() adds (callers clamp x >= 2^-126).
__device__ __forceinline__ float rsqrt_ftz(float x) {
  float y;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
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
template <bool NEWTON2 = (SDR_R_NEWTON2 != 0)>
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
#if SDR_R_SEED32
  // float32 MUFU.RSQ seed (~2^-23 vs ~2^-20 for MUFU.RSQ64H): after the one
  // Newton step r is good to ~2^-45, so ~8x fewer elements miss
  // certification; the clamp keeps k = 0 (X ~ 2^-1000) finite.
  double h = static_cast<double>(rsqrt_ftz(fmaxf(__double2float_rn(X), 0x1p-126f)));
#else
  double h = rsqrt_seed(X);
#endif
  if constexpr (NEWTON2) h = h * fma(X * h, h * -0.5, 1.5);              // seed to ~2^-45
  const double gx = X * h;
  return gx * fma(gx * h, nh, th);                                       // std * sqrt(X)
}

// cos(2*pi*k*2^-24), k = w1 >> 8: nearest pi/1024 table point + residual.
__device__ __forceinline__ double c_fast_trig(uint32_t w1, const double2* trig) {
  const double* C = c_npoly;
  const uint32_t u = w1 + 0x100000u;                                     // (k + 4096) << 8
  const double2 cs = lut_at(trig, (u >> 17) & 0x7FF0u);                  // i = u >> 21
  const double d = hilo(0x43300000u, (u >> 8) & 0x1FFFu) - kTwo52p4096;  // k - 8192 i, exact
  const double d2 = d * d;
  const double cm = d2 * fma(d2, C[4], C[5]);                            // cos(K d) - 1
  const double sd = d * fma(d2, C[6], C[7]);                             // sin(K d)
  return fma(-cs.y, sd, fma(cs.x, cm, cs.x));
}
__device__ __forceinline__ double c_fast(uint32_t w1, const NormalLut* L) { return c_fast_trig(w1, L->trig); }

// float32 fast functions for the bfloat16 path: the same reductions as
// r_fast / c_fast in float32 arithmetic (~2^-21), calibrated exhaustively like
// the float64 ones.  Tables (NormalLut32): logt[j] = (-2 mult_j 2^-23,
// 2 ln(inv_j)) (+2^-100 at j = 0), trig[i] = (cos, sin)(i pi/1024).
__device__ __forceinline__ float r32_fast(uint32_t w0, const NormalLut32* L) {
  // n = 2^24 - k by a float add (exact; one integer op less than the integer
  // subtract), e via a shift-add the compiler can fuse (LEA.HI)
  const uint32_t hw = __float_as_uint(16777216.0f - __uint2float_rn(w0 >> 8));    // n, exact
  const float2 tb = lut_at(L->logt, (hw >> 11) & 0xFF8u);                         // j = hw[22:14]
  const float s = fmaf(__uint_as_float((hw & 0x007FFFFFu) | 0x4B000000u), tb.x, 2.0f);  // -2t
  const float g = fmaf(s * s, fmaf(s, 1.0f / 12.0f, 0.25f), s);                   // -2 log1p(t)
  const float e = __uint_as_float(((hw + 0x400000u) >> 23) + 0x4B000000u) - 8388759.0f;  // e, exact
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

// Table-free float32 r for the bfloat16 path (SDR_NORMAL_BF16_MUFU):
// X = -2 ln2 lg2(w) with w = 1 - k 2^-24 exact, r = X rsqrt(X).  Two MUFU
// ops (XU pipe, beside the integer / FP32 issue) and four other instructions
// instead of r32_fast's ~15 with a bank-conflicted shared-memory load (issue
// costs: profiles/r02_issue_ubench.txt).  lg2.approx has an absolute error,
// so r's error is modelled as |r - r_np| <= Er r + Ei h, h = rsqrt(X) ~ 1/r,
// with Er, Ei measured over all 2^24 inputs at load (k_normal_calibrate_mufu);
// k = 0 clamps X to 2^-120 (h = 2^60: never certified).  It misses the
// certification about twice as often as r32_fast (0.56% vs 0.24%), which the
// per-warp miss queue (MissQ) absorbs.
__device__ __forceinline__ float r32_mufu(uint32_t w0, float& h) {
  const float w = fmaf(__uint2float_rn(w0 >> 8), -0x1p-24f, 1.0f);  // 1 - u1, exact
  float l;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(l) : "f"(w));
  const float X = fmaxf(l * -1.38629436112f, 0x1p-120f);  // -2 ln w
  h = rsqrt_ftz(X);
  return X * h;
}

// Hardware cosine of k2 2^-24 turns (cos.approx: the argument times 1/(2 pi)
// feeds MUFU.COS), absolute error Acm calibrated over all 2^24 inputs.
__device__ __forceinline__ float c32_mufu(uint32_t w1) {
  float c;
  asm("cos.approx.ftz.f32 %0, %1;" : "=f"(c) : "f"(__uint2float_rn(w1 >> 8) * 0x1.921fb6p-22f));
  return c;
}

__device__ __forceinline__ float c32_fast(uint32_t w1, const NormalLut32* L) {
  const float2 a = lut_at(L->trig_hi, (w1 >> 17) & 0x7FF8u);  // hi = k >> 12
#if SDR_C32_POLY
  // (cos, sin) of the low part d = 2 pi lo 2^-24 < 1.6e-3 by polynomial
  // instead of a second bank-conflicted table load: lo 2^8 = w1 & 0xFFF00 is
  // exact in float32, cos d = 1 - d^2/2 (next term 3e-13), sin d = d - d^3/6
  const float d = __uint2float_rn(w1 & 0x000FFF00u) * 0x1.921fb6p-30f;  // 2 pi / 2^32
  const float d2 = d * d;
  const float cl = fmaf(d2, -0.5f, 1.0f), sl = d * fmaf(d2, -0.16666667f, 1.0f);
  return fmaf(a.x, cl, -a.y * sl);
#else
  const float2 b = lut_at(L->trig_lo, (w1 >> 5) & 0x7FF8u);   // lo = k & 4095
  return fmaf(a.x, b.x, -a.y * b.y);
#endif
}

// std * r(k) from NormalLut2 (see there): s and t = s (s/2 - 2/3) in float32
// (s exact, t to 2^-24 relative), X = (A - 2s) + s^2 (1 + t) in float64, one
// Newton step on the MUFU.RSQ64H seed with std folded in (nh = -std/2,
// th = 3 std/2).  13 float64 operations fewer than r_fast + c_fast.  k = 0:
// T_0 carries 2^-1000 so X > 0 (r ~ 2^-500, never certified).
constexpr double kTwoLn2 = 0x1.62e42fefa39efp0;  // RN(2 ln 2)
__device__ __forceinline__ double r_fast2(uint32_t w0, const NormalLut2* L, double nh, double th) {
  const uint32_t hw = __float_as_uint(16777216.0f - __uint2float_rn(w0 >> 8));    // n, exact
  const LogEnt2 tb = lut_at(L->logt, (hw >> 8) & 0x7FF0u);                         // j = hw[22:12]
  const float m = __uint_as_float((hw & 0x007FFFFFu) | 0x3F800000u);
  const float s = fmaf(m, tb.inv, -1.0f);                                          // exact
  const float t = s * fmaf(s, 0.5f, -0.666666686534881591796875f);
  const double sd = static_cast<double>(s);
  // 24 - E = (2^23 + 151) - float(2^23 + biased E), exact in float32 (a
  // shift-add and an FADD instead of an integer subtract and I2F.F64)
  const float em = 8388759.0f - __uint_as_float((hw >> 23) + 0x4B000000u);
  const double A = fma(static_cast<double>(em), kTwoLn2, tb.T);                  // (24-E) 2ln2 + T_j
  const double s2 = sd * sd;                                                       // exact
  const double X = fma(sd, -2.0, A) + fma(s2, static_cast<double>(t), s2);        // -2 ln w
#if SDR_R2_SEED == 1
  // float32 MUFU.RSQ seed (~2^-23; the f64 MUFU.RSQ64H seed is ~2^-20): one
  // Newton step then leaves ~2^-45 instead of ~2^-39.5, so ~64x fewer
  // elements miss certification.  The clamp keeps k = 0 (X = 2^-1000) finite.
  const double h = static_cast<double>(rsqrt_ftz(fmaxf(__double2float_rn(X), 0x1p-126f)));
#else
  double h = rsqrt_seed(X);
#if SDR_R2_SEED == 2
  h = fma(h, 0.5 * fma(-(X * h), h, 1.0), h);  // second Newton step on 1/sqrt(X)
#endif
#endif
  const double gx = X * h;
  return gx * fma(gx * h, nh, th);                                                 // std * sqrt(X)
}

// cos(2*pi*k2*2^-24), k2 = w1 >> 8.  SDR_N2_COS2: two-level table, k2 =
// 4096 i + b, C_i C_b - S_i S_b (2 float64 ops, 32 B of random shared-memory
// reads); else c_fast's pi/1024 table + residual polynomial (16 B, 8 ops).
// Random 16 B shared loads cost ~12 wavefronts per warp (bank conflicts), so
// the bytes per element bound the kernel as much as the float64 ops do.
__device__ __forceinline__ double c_fast2(uint32_t w1, const NormalLut2* L) {
#if SDR_N2_COS2
  const double2 a = lut_at(L->cos_hi, (w1 >> 16) & 0xFFF0u);
  const double2 b = lut_at(L->cos_lo, (w1 >> 4) & 0xFFF0u);
  return fma(a.x, b.x, -(a.y * b.y));
#else
  return c_fast_trig(w1, L->trig);
#endif
}

template <int DT>
__device__ __forceinline__ typename St<DT>::T normal_value(const DistP& P, const NormalLut* L,
                                                           uint32_t w0, uint32_t w1);

// Per-warp queue of the bfloat16 elements the float32 path could not
// certify (~0.24% of them).  Resolving one inline costs a whole divergent
// float64 evaluation with one lane active (measured: ~12% of a fill, ~17% of
// the LLaMA-3-8B init); queued, they are resolved by the converged warp, one
// element per lane (missq_flush at the end of a kernel / of a batch tile).
// The queued element's slot already holds a placeholder from the chunk's
// vector store; the flush overwrites it after a __syncwarp (memory order
// between the warp's threads).  A full queue falls back to the inline path.
#ifndef SDR_F32_XORCERT
#define SDR_F32_XORCERT 1  // float32 / float16 certification by XOR-accumulate (else per-element compare; 1.5-2.5% slower)
#endif
#ifndef SDR_MISSQ_N
#define SDR_MISSQ_N 256
#endif
constexpr int kMissQ = SDR_MISSQ_N;
struct MissQ {
  uint4 e[kMissQ];  // (address lo, address hi, w0, w1)
  uint32_t n;
};
__device__ __forceinline__ MissQ* missq() {
  __shared__ MissQ s_mq[256 / 32];  // one per warp of a 256-thread CTA (the bfloat16 fill kernels)
  return &s_mq[threadIdx.x >> 5];
}
__device__ __forceinline__ void missq_init() {
  if ((threadIdx.x & 31) == 0) missq()->n = 0;
  __syncwarp();
}

// A chunk of bfloat16 normals on the float32 path.  Elements go in pairs: one
// F2FP packs the two lower ends RD(v - B) and one the two upper ends RU(v + B)
// (bf16(RN32(.)) is monotone, so an element is certified iff both ends round
// to the same bfloat16); the lower pack is the output word, and the XOR of the
// two packs is OR-accumulated (one LOP3 per pair).  Only the rare branch looks
// at which element differs; those take the float64 path, then the exact one.
template <int DT, int NE>
__device__ __forceinline__ void normal_chunk_bf16(const DistP& P, const NormalLut32* L32,
                                                  const uint32_t* w0, const uint32_t* w1, uint16_t* out,
                                                  uint16_t* qdst = nullptr, int nvalid = NE) {
  static_assert(NE % 2 == 0, "elements go in pairs");
  uint32_t diff = 0, hiw[NE / 2];
#pragma unroll
  for (int e = 0; e < NE; e += 2) {
    float lo[2], hi[2];
#pragma unroll
    for (int i = 0; i < 2; ++i) {
#if SDR_NORMAL_BF16_MUFU
      float h;
      float r, c, B;
      if constexpr (cos_mufu<DT>()) {
        r = r32_mufu(w0[e + i], h);
        c = c32_mufu(w1[e + i]);
        B = fmaf(h, P.nm.bmc_i, fmaf(r, P.nm.bmc_r, P.nm.bm_c));
      } else {
        r = r32_mufu(w0[e + i], h);
        c = c32_fast(w1[e + i], L32);
        // |v - v_numpy| <= r*bm_r + h*bm_i + bm_c   (host: fill_dist_params)
        B = fmaf(h, P.nm.bm_i, fmaf(r, P.nm.bm_r, P.nm.bm_c));
      }
      const float v = fmaf(P.nm.std32, r * c, P.nm.mean32);
#else
      const float r = r32_fast(w0[e + i], L32), c = c32_fast(w1[e + i], L32);
      const float v = fmaf(P.nm.std32, r * c, P.nm.mean32);
      // |v - v_numpy| <= r*b32_r + b32_c   (host: bound terms; |v| term folded)
      const float B = fmaf(r, P.nm.b32_r, P.nm.b32_c);
#endif
      lo[i] = __fsub_rd(v, B);
      hi[i] = __fadd_ru(v, B);
    }
    uint32_t l32, h32;
    if constexpr (DT == SDR_BF16) {
      const __nv_bfloat162 pl = __floats2bfloat162_rn(lo[0], lo[1]), ph = __floats2bfloat162_rn(hi[0], hi[1]);
      memcpy(&l32, &pl, 4);
      memcpy(&h32, &ph, 4);
    } else {  // float16: the same monotone-rounding argument with its packed conversion
      const __half2 pl = __floats2half2_rn(lo[0], lo[1]), ph = __floats2half2_rn(hi[0], hi[1]);
      memcpy(&l32, &pl, 4);
      memcpy(&h32, &ph, 4);
    }
    out[e] = static_cast<uint16_t>(l32);  // (copying the packed word whole measured 3% slower)
    out[e + 1] = static_cast<uint16_t>(l32 >> 16);
    diff |= l32 ^ h32;
    hiw[e / 2] = h32;
  }
  if (__builtin_expect(diff != 0, 0)) {
#pragma unroll
    for (int e = 0; e < NE; ++e) {
      if (e < nvalid && out[e] != static_cast<uint16_t>(hiw[e / 2] >> (16 * (e & 1)))) {
#if SDR_COUNT_F32_MISS
        atomicAdd(P.nm.fallbacks, 1ull);
#endif
#if SDR_MISSQ
        if (qdst != nullptr) {  // queue it (qdst = this chunk's destination in global memory)
          MissQ* q = missq();
          const uint32_t pos = atomicAdd(&q->n, 1u);
          if (pos < kMissQ) {
            const uint64_t a = reinterpret_cast<uint64_t>(qdst + e);
            q->e[pos] = make_uint4(static_cast<uint32_t>(a), static_cast<uint32_t>(a >> 32), w0[e], w1[e]);
            continue;
          }
        }
#endif
        // float64 certified path (tables read through L1/L2), then the exact mirror
        out[e] = normal_value<DT>(P, P.nm.lut, w0[e], w1[e]);
      }
    }
  }
}

// Resolve the warp's queued elements: the float64 certified path (tables
// through L1), then the exact mirror, one element per lane.  The whole warp
// must be converged here.
template <int DT>
__device__ __noinline__ void missq_flush(const DistP& P) {
  MissQ* q = missq();
  __syncwarp();
  const uint32_t n = min(q->n, static_cast<uint32_t>(kMissQ));
  for (uint32_t k = threadIdx.x & 31; k < n; k += 32) {
    const uint4 t = q->e[k];
    const uint16_t v = normal_value<DT>(P, P.nm.lut, t.z, t.w);
    *reinterpret_cast<uint16_t*>((static_cast<uint64_t>(t.y) << 32) | t.x) = v;
  }
  __syncwarp();
  if ((threadIdx.x & 31) == 0) q->n = 0;
  __syncwarp();
}

// CUDA libm value d of table point k corrected to NumPy's (ExactMirror).
__device__ __noinline__ double mirror_fix(double d, const uint32_t* code, uint32_t k, const uint32_t* xk,
                                          const double* xv, int32_t nx) {
  const uint32_t c = (__ldg(code + (k >> 4)) >> ((k & 15u) * 2u)) & 3u;
  if (c == 3u) {  // exception: binary search of the sorted keys
    int lo = 0, hi = nx - 1;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (__ldg(xk + mid) < k) lo = mid + 1;
      else hi = mid;
    }
    return __ldg(xv + lo);
  }
  const long long b = __double_as_longlong(d);
  return c == 0u ? d : __longlong_as_double(c == 1u ? b + 1 : b - 1);
}

// NumPy's r[k1] and c[k2] (rng.py:154-155): the device's log1p / cos of the
// same float64 arguments, corrected by the mirror; sqrt is correctly rounded.
__device__ __forceinline__ double mirror_r(const ExactMirror& M, uint32_t k) {
  const double L = mirror_fix(log1p(-static_cast<double>(k) * 0x1p-24), M.code_l, k, M.xk_l, M.xv_l, M.nx_l);
  return __dsqrt_rn(-2.0 * L);
}
__device__ __forceinline__ double mirror_c(const ExactMirror& M, uint32_t k) {
  const double arg = __dmul_rn(6.283185307179586, static_cast<double>(k) * 0x1p-24);  // (2.0*pi)*u2
  return mirror_fix(cos(arg), M.code_c, k, M.xk_c, M.xv_c, M.nx_c);
}

// Exact Normal (rng.py:150-156): float64 Box-Muller with the reference's own
// r[k1], c[k2] (compact mirror, or the full tables if it failed verification),
// then one cast.
template <int DT>
__device__ __noinline__ typename St<DT>::T normal_exact(const DistP& P, uint32_t w0, uint32_t w1) {
  double r, c;
  if (P.nm.rtab != nullptr) {
    r = __ldg(P.nm.rtab + (w0 >> 8));
    c = __ldg(P.nm.ctab + (w1 >> 8));
  } else {
    r = mirror_r(P.nm.em, w0 >> 8);
    c = mirror_c(P.nm.em, w1 >> 8);
  }
  return from_f64<DT>(__dadd_rn(P.mean, __dmul_rn(P.stdv, __dmul_rn(r, c))));
}

// float64 outputs: NumPy's r[k] and c[k] bit for bit as the fast functions
// (r_unit, c_fast) plus a signed correction of their bit patterns per table
// point, dr[k] = bits(r_np[k]) - bits(r_unit(k)) (8 bits, SDR_F64_R8) and
// dc[k] likewise (16 bits): 48 MiB per device.  Built and checked against the verified
// mirror on all 2^24 points at load (k_normal_deltas); kDeltaEsc marks the
// points whose difference does not fit (k = 0 for r, the cosine next to its
// zeros), which take the mirror.  Replaces two libm calls, a square root and
// two code lookups per element by ~25 float64 operations and two 2-byte loads
// that hit L2.
constexpr int kDeltaEsc = -32768;
// r with std = 1 as the corrections are taken against
__device__ __forceinline__ double r_unit(uint32_t w0, const NormalLut* L) {
  return r_fast<SDR_F64_R8 != 0>(w0, L, -0.5, 1.5);
}
__device__ __forceinline__ double apply_delta(double a, int d) {
  return __longlong_as_double(__double_as_longlong(a) + d);
}
#ifndef SDR_DELTA_EVICT_LAST
#define SDR_DELTA_EVICT_LAST 1  // correction loads keep their lines in L2 (evict_last), no L1 allocation
#endif
__device__ __forceinline__ uint64_t delta_policy() {
  uint64_t pol = 0;
#if SDR_DELTA_EVICT_LAST
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
#endif
  return pol;
}
__device__ __forceinline__ int ld_delta(const int16_t* p, uint64_t pol) {
#if SDR_DELTA_EVICT_LAST
  short v;
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.b16 %0, [%1], %2;" : "=h"(v) : "l"(p), "l"(pol));
  return v;
#else
  (void)pol;
  return __ldg(p);
#endif
}
__device__ __forceinline__ int ld_delta(const int8_t* p, uint64_t pol) {
#if SDR_DELTA_EVICT_LAST
  int v;
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.s8 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
  return v;
#else
  (void)pol;
  return __ldg(p);
#endif
}
// NumPy's cosine argument (rng.py:155) and cos of it in double-double; the
// result is RN(c) and `flag` marks the elements c_cr cannot vouch for.  T is
// M.cdd or its copy in shared memory.
__device__ __forceinline__ double c_cr(uint32_t w1, const CosDD* T, bool& flag) {
  const uint32_t k = w1 >> 8;
  const double u = hilo(0x43300000u - (24u << 20), k) - 0x1p28;            // k 2^-24, exact
  const double arg = __dmul_rn(6.283185307179586, u);                     // (2.0 * pi) * u2
  const uint32_t i = (k + 4096u) >> 13;                                    // nearest i pi/1024
  const double fi = hilo(0x43300000u, i) - 0x1p52;
  const double d1 = fma(-fi, kQ1, arg);                                   // exact
  const double p2 = fi * kQ2;                                             // exact
  const double dh = d1 - p2;                                               // TwoSum
  const double bb = dh - d1;
  const double dl = fma(-fi, kQ3, (d1 - (dh - bb)) + (-p2 - bb));         // d = dh + dl
  const CosDD t = T[i];
  const double ph = dh * dh;
  const double pl = fma(dh, dh, -ph) + 2.0 * dh * dl;                      // d^2 = ph + pl
  const double cmh = -0.5 * ph;                                            // cos d - 1 = cmh + cml
  const double cml = fma(-0.5, pl, ph * ph * fma(ph, -1.0 / 720.0, 1.0 / 24.0));
  const double sdl = fma(dh * ph, fma(ph, 1.0 / 120.0, -1.0 / 6.0), dl);   // sin d = dh + sdl
  // c = C (1 + cm) - S sin d
  const double t1 = t.sh * dh, e1 = fma(t.sh, dh, -t1);
  const double t2 = t.ch * cmh, e2 = fma(t.ch, cmh, -t2);
  const double s1 = t.ch - t1, b1 = s1 - t.ch, r1 = (t.ch - (s1 - b1)) + (-t1 - b1);
  const double s2 = s1 + t2, b2 = s2 - s1, r2 = (s1 - (s2 - b2)) + (t2 - b2);
  double lo = (r1 + r2) + ((e2 - e1) + t.cl);
  lo = fma(-t.sh, sdl, lo);
  lo = fma(-t.sl, dh, lo);
  lo = fma(t.ch, cml, lo);
  lo = fma(t.cl, cmh, lo);
  const double c = s2 + lo;
  const double rem = lo - (c - s2);                                        // exact: c + rem
  const uint32_t hw = dhi(c), ex = hw & 0x7FF00000u;
  const double ulp = hilo(ex - (52u << 20), 0u);
  flag = ex < ((1023u - 10u) << 20) || (dlo(c) == 0u && (hw & 0xFFFFFu) == 0u) ||
         fabs(fabs(rem) - 0.5 * ulp) < SDR_COS_TAU * ulp;
  return c;
}

__device__ __forceinline__ const int8_t* dc8(const NormalMirror& M) {
  return reinterpret_cast<const int8_t*>(M.dr) + (sizeof(DeltaR) << 24);
}

__device__ __forceinline__ double normal_f64_of(const DistP& P, double r, double c) {
  return __dadd_rn(P.mean, __dmul_rn(P.stdv, __dmul_rn(r, c)));  // rng.py:156, as normal_exact
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
  if constexpr (DT == SDR_F64) {
    if (P.nm.dr != nullptr) {
      const int dr = __ldg(P.nm.dr + (w0 >> 8));
      if (P.nm.cdd != nullptr) {
        bool flag;
        double c = c_cr(w1, P.nm.cdd, flag);
        int dc = 0;
        if (flag) dc = __ldg(dc8(P.nm) + (w1 >> 8));
        if (dr != kDeltaEscR && dc != -128) return normal_f64_of(P, apply_delta(r_unit(w0, L), dr), apply_delta(c, dc));
      } else {
        const int dc = __ldg(P.nm.dc + (w1 >> 8));
        if (dr != kDeltaEscR && dc != kDeltaEsc)
          return normal_f64_of(P, apply_delta(r_unit(w0, L), dr), apply_delta(c_fast(w1, L), dc));
      }
    }
  } else {
    bool ok;
    const auto v = normal_certified<DT>(P, r_fast(w0, L, P.nm.nh, P.nm.th), c_fast(w1, L), ok);
    if (__builtin_expect(ok, 1)) return v;
    atomicAdd(P.nm.fallbacks, 1ull);
  }
  return normal_exact<DT>(P, w0, w1);
}

// A chunk of float64 normals from the per-point corrections: the 2-byte loads
// first (their L2 latency overlaps the float64 work), then all r, all c, then
// the reference's three roundings; one branch for the rare escapes.
template <int NE>
__device__ __forceinline__ void normal_chunk_f64(const DistP& P, const NormalLut* L, const uint32_t* w0,
                                                 const uint32_t* w1, double* out) {
  if (P.nm.dr == nullptr) {
#pragma unroll
    for (int e = 0; e < NE; ++e) out[e] = normal_exact<SDR_F64>(P, w0[e], w1[e]);
    return;
  }
  int dr[NE], dc[NE];
  const uint64_t pol = delta_policy();
  double r[NE], c[NE];
  bool esc = false;
  const bool cr = P.nm.cdd != nullptr;
  if (cr) {
    // the cosine from c_cr: only its flagged elements (a few percent) read a correction
#pragma unroll
    for (int e = 0; e < NE; ++e) dr[e] = ld_delta(P.nm.dr + (w0[e] >> 8), pol);
    bool flag[NE];
    const CosDD* T = P.nm.cdd;  // 64 KiB, through L1 (prefer_l1)
#pragma unroll
    for (int e = 0; e < NE; ++e) c[e] = c_cr(w1[e], T, flag[e]);
#pragma unroll
    for (int e = 0; e < NE; ++e) dc[e] = flag[e] ? ld_delta(dc8(P.nm) + (w1[e] >> 8), pol) : 0;
#pragma unroll
    for (int e = 0; e < NE; ++e) r[e] = r_unit(w0[e], L);
#pragma unroll
    for (int e = 0; e < NE; ++e) esc |= (dr[e] == kDeltaEscR) | (dc[e] == -128);
  } else {
#pragma unroll
    for (int e = 0; e < NE; ++e) {
      dr[e] = ld_delta(P.nm.dr + (w0[e] >> 8), pol);
      dc[e] = ld_delta(P.nm.dc + (w1[e] >> 8), pol);
    }
#pragma unroll
    for (int e = 0; e < NE; ++e) r[e] = r_unit(w0[e], L);
#pragma unroll
    for (int e = 0; e < NE; ++e) c[e] = c_fast(w1[e], L);
#pragma unroll
    for (int e = 0; e < NE; ++e) esc |= (dr[e] == kDeltaEscR) | (dc[e] == kDeltaEsc);
  }
#pragma unroll
  for (int e = 0; e < NE; ++e) out[e] = normal_f64_of(P, apply_delta(r[e], dr[e]), apply_delta(c[e], dc[e]));
  if (__builtin_expect(esc, 0)) {
#pragma unroll
    for (int e = 0; e < NE; ++e)
      if (dr[e] == kDeltaEscR || dc[e] == (cr ? -128 : kDeltaEsc))
        out[e] = normal_exact<SDR_F64>(P, w0[e], w1[e]);
  }
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
#if SDR_F32_XORCERT
  // the XOR of the two roundings OR-accumulated (one LOP3 per element); the
  // rare branch finds the differing elements
  using T = typename St<DT>::T;
  uint32_t diff = 0;
  T hib[NE];
#pragma unroll
  for (int e = 0; e < NE; ++e) {
    const double v = fma(rs[e], c[e], P.mean);
    const double B = fma(rs[e], P.nm.kr, P.nm.k0);
    const T lo = from_f64<DT>(v - B), hi = from_f64<DT>(v + B);
    out[e] = lo;
    hib[e] = hi;
    if constexpr (DT == SDR_F32) diff |= __float_as_uint(lo) ^ __float_as_uint(hi);
    else diff |= static_cast<uint32_t>(lo ^ hi);
  }
  if (__builtin_expect(diff != 0, 0)) {
#pragma unroll
    for (int e = 0; e < NE; ++e) {
      bool same;
      if constexpr (DT == SDR_F32) same = __float_as_uint(out[e]) == __float_as_uint(hib[e]);
      else same = out[e] == hib[e];
      if (!same) {
        atomicAdd(P.nm.fallbacks, 1ull);
        out[e] = normal_exact<DT>(P, w0[e], w1[e]);
      }
    }
  }
#else
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
#endif
}
// A chunk of float32 / float16 normals on the NormalLut2 tables: all r, all c,
// combine, certify by rounding v - B and v + B (the cast is monotone), one
// branch for the rare uncertified elements (exact NumPy mirror).  The
// certification test costs one LOP3 per element: the XOR of the two roundings
// is OR-accumulated over the chunk, and only the rare branch looks at which
// element differs.
template <int DT, int NE>
__device__ __forceinline__ void normal_chunk2(const DistP& P, const NormalLut2* L, const uint32_t* w0,
                                              const uint32_t* w1, typename St<DT>::T* out) {
  using T = typename St<DT>::T;
  double rs[NE], c[NE];
#pragma unroll
  for (int e = 0; e < NE; ++e) rs[e] = r_fast2(w0[e], L, P.nm.nh, P.nm.th);
#pragma unroll
  for (int e = 0; e < NE; ++e) c[e] = c_fast2(w1[e], L);
  uint32_t diff = 0;
  T hib[NE];
#pragma unroll
  for (int e = 0; e < NE; ++e) {
    const double v = fma(rs[e], c[e], P.mean);
    const double B = fma(rs[e], P.nm.kr2, P.nm.k02);
    const T lo = from_f64<DT>(v - B), hi = from_f64<DT>(v + B);
    out[e] = lo;
    hib[e] = hi;
    uint32_t a, b;
    if constexpr (DT == SDR_F32) {
      a = __float_as_uint(lo);
      b = __float_as_uint(hi);
    } else {
      a = lo;
      b = hi;
    }
    diff |= a ^ b;
  }
  if (__builtin_expect(diff != 0, 0)) {
#pragma unroll
    for (int e = 0; e < NE; ++e) {
      bool same;
      if constexpr (DT == SDR_F32) same = __float_as_uint(out[e]) == __float_as_uint(hib[e]);
      else same = out[e] == hib[e];
      if (!same) {
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
