// dropout.cu -- fused sharded dropout for sm_100a: the keep-mask of
// Bernoulli(1-p) drawn from the shared Philox stream over this rank's window
// (rng.py:238-242, dispatch.py:567-576) applied as y = (x*m)*(1/(1-p))
// (engine.py:80-81) in one kernel; the mask is optional (the backward
// regenerates it).  Only w1 of each Philox block decides keep, except on the
// 2^-32 tie (see k_dropout_fast).
#include <cmath>
#include <cstring>

#include "rng_common.cuh"

namespace sdr {

// ---------------------------------------------------------------------------
// Fused dropout: y = (x*m)*scale, m from Bernoulli(1-p) (engine.py:80-81).
// ---------------------------------------------------------------------------
struct DropArgs {
  Gen g;
  ViewIndexer ix;
  const void* x;
  void* y;
  void* mask;
  uint64_t keep_le;   // keep <=> (w1:w0) <= keep_le, i.e. k53 < ceil((1-p)*2^53)
  uint32_t aligned;   // THETA pow2 >= chunk and every chunk start chunk-aligned
  float scale32;
  double scale64;
  uint16_t scale16;  // f16 bits of the scale
  uint32_t ragged;   // inner extent not a multiple of the chunk: k_dropout_ragged
  uint64_t nchunks;
  uint64_t chunks_per_row;
  FastDiv64 div_cpr;
};

template <int XT> struct DropT { using T = typename St<XT>::T; };

// y element for input dtype XT and output dtype YT; sets `nan` when the
// result is a NaN (then drop_nan_fix() supplies the x86/NumPy bit pattern).
template <int XT, int YT>
__device__ __forceinline__ typename St<YT>::T drop_apply(const DropArgs& A, typename St<XT>::T x,
                                                         bool keep, bool& nan) {
  // (x * m) * scale == x * (m ? scale : 0) bit for bit: x * 1 is exact, and
  // (x * 0) * scale == x * 0 (a signed zero, or NaN for NaN / inf x) since the
  // float32 / float64 scale is positive and finite (1/(1-p) <= 2^53 for any
  // double p < 1) -- one multiply per element less.
  if constexpr (XT == SDR_F32) {
    const float y = __fmul_rn(x, keep ? A.scale32 : 0.0f);
    nan = y != y;
    return y;
  } else if constexpr (XT == SDR_F64) {
    const double y = __dmul_rn(x, keep ? A.scale64 : 0.0);
    nan = y != y;
    return y;
  } else if constexpr (XT == SDR_BF16) {
    const float xf = __uint_as_float(static_cast<uint32_t>(x) << 16);
    const float y = __fmul_rn(xf, keep ? A.scale32 : 0.0f);
    nan = y != y;
    if constexpr (YT == SDR_F32) return y;
    else return bf16_bits(y);
  } else {  // SDR_F16: x*m exact in f16, then RNE(x16 * scale16)
    const __half xh = __ushort_as_half(x);
    // (no folding here: scale16 overflows to inf for p > 1 - 2^-16, and (x * 0) * inf is NaN)
    const __half xm = __hmul(xh, keep ? __ushort_as_half(0x3C00) : __ushort_as_half(0));
    const uint16_t y = __half_as_ushort(__hmul(xm, __ushort_as_half(A.scale16)));
    nan = (y & 0x7FFFu) > 0x7C00u;
    return y;
  }
}

// NaN results as x86 SSE + NumPy / ml_dtypes produce them: a NaN input is
// propagated quieted with its payload, inf*0 gives the negative default NaN;
// float32->bfloat16 maps NaN to 0x7FC0 / 0xFFC0 (ml_dtypes), float->half keeps
// sign and the top payload bits (numpy npy_floatbits_to_halfbits).
template <int XT, int YT>
__device__ __noinline__ typename St<YT>::T drop_nan_fix(typename St<XT>::T x) {
  if constexpr (XT == SDR_F32) {
    const uint32_t b = __float_as_uint(x);
    return __uint_as_float((b & 0x7FFFFFFFu) > 0x7F800000u ? (b | 0x00400000u) : 0xFFC00000u);
  } else if constexpr (XT == SDR_F64) {
    const uint64_t b = static_cast<uint64_t>(__double_as_longlong(x));
    const bool isn = (b & 0x7FFFFFFFFFFFFFFFull) > 0x7FF0000000000000ull;
    return __longlong_as_double(static_cast<long long>(isn ? (b | 0x0008000000000000ull)
                                                           : 0xFFF8000000000000ull));
  } else if constexpr (XT == SDR_BF16) {
    const uint32_t b = static_cast<uint32_t>(x) << 16;
    const uint32_t f = (b & 0x7FFFFFFFu) > 0x7F800000u ? (b | 0x00400000u) : 0xFFC00000u;
    if constexpr (YT == SDR_F32) return __uint_as_float(f);
    else return static_cast<uint16_t>((f & 0x80000000u) ? 0xFFC0u : 0x7FC0u);
  } else {
    const uint16_t b = x;
    return static_cast<uint16_t>((b & 0x7FFFu) > 0x7C00u ? (b | 0x0200u) : 0xFE00u);
  }
}

#ifndef SDR_DROP_MINB
#define SDR_DROP_MINB 4
#endif
#ifndef SDR_DROP_SPLIT
#define SDR_DROP_SPLIT 1   // Philox for the chunk in SPLIT passes
#endif
#ifndef SDR_DROP_CH
#define SDR_DROP_CH 8      // elements per thread-chunk of the dropout kernel
#endif
constexpr int kDropCh = SDR_DROP_CH;

__device__ __forceinline__ uint64_t drop_chunk_base(const DropArgs& A, uint64_t q) {
  const CanonView& cv = A.ix.cv;
  if (cv.nd == 0) return static_cast<uint64_t>(cv.base) + q * kDropCh;  // one contiguous run
  return outer_base(A.ix, A.div_cpr, q, kDropCh);
}


// bf16 lanes of a 32-bit word as float32 (PRMT / LOP3 on the ALU pipe).
__device__ __forceinline__ float bf16_lo(uint32_t w) { return __uint_as_float(__byte_perm(w, 0u, 0x1044)); }
__device__ __forceinline__ float bf16_hi(uint32_t w) { return __uint_as_float(w & 0xFFFF0000u); }

// y = (x*m)*scale for one chunk given its keep flags; NaN fix-up; stores y
// (and the mask when requested).
template <int XT, int YT, int MT, int CH>
__device__ __forceinline__ void drop_store(const DropArgs& A, uint64_t q,
                                           const typename St<XT>::T (&xv)[CH], const bool (&keep)[CH]) {
  using XTy = typename St<XT>::T;
  using YTy = typename St<YT>::T;
  YTy yv[CH];
  bool anynan = false, nan[CH];
#pragma unroll
  for (int e = 0; e < CH; ++e) {
    if constexpr (XT == SDR_BF16) {
      uint32_t wd;
      memcpy(&wd, &xv[e & ~1], 4);
      const float xf = (e & 1) ? bf16_hi(wd) : bf16_lo(wd);
      const float r = __fmul_rn(__fmul_rn(xf, keep[e] ? 1.0f : 0.0f), A.scale32);
      nan[e] = r != r;
      if constexpr (YT == SDR_F32) yv[e] = r;
      else yv[e] = bf16_bits(r);
    } else {
      yv[e] = drop_apply<XT, YT>(A, xv[e], keep[e], nan[e]);
    }
    anynan |= nan[e];
  }
  if (anynan) {
#pragma unroll
    for (int e = 0; e < CH; ++e)
      if (nan[e]) yv[e] = drop_nan_fix<XT, YT>(xv[e]);
  }
  store_chunk(static_cast<YTy*>(A.y) + q * CH, yv);
  if constexpr (MT >= 0) {
    using MTy = typename St<MT>::T;
    if (A.mask != nullptr) {
      MTy mv[CH];
#pragma unroll
      for (int e = 0; e < CH; ++e) mv[e] = one_or_zero<MT>(keep[e]);
      store_chunk(static_cast<MTy*>(A.mask) + q * CH, mv);
    }
  }
}

template <int XT, int YT, int MT, bool ALIGNED>
__global__ void __launch_bounds__(256, SDR_DROP_MINB) k_dropout_fast(const __grid_constant__ DropArgs A) {
  using XTy = typename St<XT>::T;
  using YTy = typename St<YT>::T;
  const XTy* x = static_cast<const XTy*>(A.x);
  YTy* y = static_cast<YTy*>(A.y);
  constexpr int CH = kDropCh;
  constexpr int NE = CH / SDR_DROP_SPLIT;
#if SDR_PDL
  // Programmatic dependent launch: let the next kernel on the stream start its
  // CTAs as ours drain, and wait here until the previous grid's memory is
  // visible (a no-op when launched without the attribute).
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
#endif
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t q = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; q < A.nchunks;
       q += stride) {
    XTy xv[CH];
    load_chunk(x + q * CH, xv);
    const uint64_t j0 = drop_chunk_base(A, q);  // (an incremental walk measured slower here)
    YTy yv[CH];
    bool keep[CH], anynan = false, nan[CH];
#pragma unroll
    for (int h = 0; h < SDR_DROP_SPLIT; ++h) {
      uint32_t w0[NE], w1[NE];
      if constexpr (ALIGNED) {
        chunk_w1_aligned<NE>(A.g, j0 + h * NE, w1);
      } else {
        chunk_words<NE>(A.g, j0 + h * NE, w0, w1);
      }
#pragma unroll
      for (int i = 0; i < NE; ++i) {
        const int e = h * NE + i;
        if constexpr (ALIGNED) {
          // (w1:w0) <= keep_le is decided by w1 unless w1 equals its high word
          // (p = 2^-32): per-element rare branch (measured faster than one
          // merged branch per chunk)
          const uint32_t H = hi32(A.keep_le);
          keep[e] = w1[i] < H;
          if (__builtin_expect(w1[i] == H, 0)) {
            uint32_t f0, f1;
            elem_words(A.g, j0 + e, f0, f1);
            keep[e] = ((static_cast<uint64_t>(f1) << 32) | f0) <= A.keep_le;
          }
        }
        if constexpr (!ALIGNED) {
          const uint64_t u64 = (static_cast<uint64_t>(w1[i]) << 32) | w0[i];
          keep[e] = u64 <= A.keep_le;
        }
        if constexpr (XT == SDR_BF16) {
          // unpack from the raw 16 B vector: even lane = low half of a word
          uint32_t wd;
          memcpy(&wd, &xv[e & ~1], 4);
          const float xf = (e & 1) ? bf16_hi(wd) : bf16_lo(wd);
          const float r = __fmul_rn(xf, keep[e] ? A.scale32 : 0.0f);  // == (x * m) * scale (drop_apply)
          nan[e] = r != r;
          if constexpr (YT == SDR_F32) yv[e] = r;
          else yv[e] = bf16_bits(r);
        } else {
          yv[e] = drop_apply<XT, YT>(A, xv[e], keep[e], nan[e]);
        }
        anynan |= nan[e];
      }
    }
    if (anynan) {
#pragma unroll
      for (int e = 0; e < CH; ++e)
        if (nan[e]) yv[e] = drop_nan_fix<XT, YT>(xv[e]);
    }
    store_chunk(y + q * CH, yv);
    if constexpr (MT >= 0) {
      using MTy = typename St<MT>::T;
      if (A.mask != nullptr) {
        MTy mv[CH];
#pragma unroll
        for (int e = 0; e < CH; ++e) mv[e] = one_or_zero<MT>(keep[e]);
        store_chunk(static_cast<MTy*>(A.mask) + q * CH, mv);
      }
    }
  }
}

// Ragged rows (inner extent not a multiple of the chunk): chunk q = (row, cq)
// covers columns [CH cq, min(CH cq + CH, inner)) of its row.  Philox is
// computed CH-wide on consecutive global indices (hoisted rounds 1-2), x / y /
// mask move per element (row starts are not 16 B aligned).
template <int XT, int YT, int MT>
__global__ void __launch_bounds__(256) k_dropout_ragged(const __grid_constant__ DropArgs A) {
  using XTy = typename St<XT>::T;
  using YTy = typename St<YT>::T;
  constexpr int CH = kDropCh;
  const XTy* x = static_cast<const XTy*>(A.x);
  YTy* y = static_cast<YTy*>(A.y);
  const CanonView& cv = A.ix.cv;
  const uint64_t inner = static_cast<uint64_t>(cv.inner);
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t q = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; q < A.nchunks;
       q += stride) {
    uint64_t row, cq;
    A.div_cpr.divmod(q, row, cq);
    uint64_t j0 = static_cast<uint64_t>(cv.base) + cq * CH, r = row;
    for (int k = cv.nd - 1; k >= 1; --k) {
      uint64_t qq, rem;
      A.ix.div_o[k].divmod(r, qq, rem);
      j0 += rem * static_cast<uint64_t>(cv.ostride[k]);
      r = qq;
    }
    if (cv.nd >= 1) j0 += r * static_cast<uint64_t>(cv.ostride[0]);
    const uint64_t lq = row * inner + cq * CH;
    const int nvalid = static_cast<int>(min(static_cast<uint64_t>(CH), inner - cq * CH));
    uint32_t w0[CH], w1[CH];
    chunk_words<CH>(A.g, j0, w0, w1);
#pragma unroll
    for (int e = 0; e < CH; ++e) {
      if (e < nvalid) {
        const uint64_t i = lq + e;
        const bool keep = ((static_cast<uint64_t>(w1[e]) << 32) | w0[e]) <= A.keep_le;
        bool nan;
        const XTy xe = x[i];
        const YTy v = drop_apply<XT, YT>(A, xe, keep, nan);
        y[i] = nan ? drop_nan_fix<XT, YT>(xe) : v;
        if constexpr (MT >= 0) {
          using MTy = typename St<MT>::T;
          if (A.mask != nullptr) static_cast<MTy*>(A.mask)[i] = one_or_zero<MT>(keep);
        }
      }
    }
  }
}

template <int XT, int YT, int MT>
__global__ void __launch_bounds__(256) k_dropout_generic(const __grid_constant__ DropArgs A) {
  using XTy = typename St<XT>::T;
  using YTy = typename St<YT>::T;
  const XTy* x = static_cast<const XTy*>(A.x);
  YTy* y = static_cast<YTy*>(A.y);
  const uint64_t n = static_cast<uint64_t>(A.ix.cv.numel);
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += stride) {
    uint32_t w0, w1;
    elem_words(A.g, A.ix.global_of(i), w0, w1);
    const uint64_t u64 = (static_cast<uint64_t>(w1) << 32) | w0;
    const bool keep = u64 <= A.keep_le;
    bool nan;
    const YTy v = drop_apply<XT, YT>(A, x[i], keep, nan);
    y[i] = nan ? drop_nan_fix<XT, YT>(x[i]) : v;
    if constexpr (MT >= 0) {
      using MTy = typename St<MT>::T;
      if (A.mask != nullptr) static_cast<MTy*>(A.mask)[i] = one_or_zero<MT>(keep);
    }
  }
}

template <int XT, int YT, int MT>
static int launch_drop(const DropArgs& A, bool fast, cudaStream_t s) {
  if (A.ragged)
    k_dropout_ragged<XT, YT, MT><<<grid_for(k_dropout_ragged<XT, YT, MT>, A.nchunks, 256), 256, 0, s>>>(A);
  else if (fast && A.aligned)
    launch_pdl(k_dropout_fast<XT, YT, MT, true>, grid_for(k_dropout_fast<XT, YT, MT, true>, A.nchunks, 256), s, A);
  else if (fast)
    launch_pdl(k_dropout_fast<XT, YT, MT, false>, grid_for(k_dropout_fast<XT, YT, MT, false>, A.nchunks, 256), s, A);
  else
    k_dropout_generic<XT, YT, MT><<<grid_for(k_dropout_generic<XT, YT, MT>, A.ix.cv.numel, 256), 256, 0, s>>>(A);
  return check_launch();
}

template <int XT, int YT>
static int dispatch_drop_mask(int mt, const DropArgs& A, bool fast, cudaStream_t s) {
  if (A.mask == nullptr) return launch_drop<XT, YT, -1>(A, fast, s);
  if (mt == SDR_U8 || mt == SDR_BOOL) return launch_drop<XT, YT, SDR_U8>(A, fast, s);
  if (mt == XT) return launch_drop<XT, YT, XT>(A, fast, s);
  return SDR_E_DTYPE;
}

int dropout(const void* x, int xt, void* y, int yt, void* mask, int mt, double p,
            const sdr_rng& rng, const sdr_view& view, cudaStream_t s) {
  if (!(p >= 0.0 && p < 1.0)) return SDR_E_PARAM;
  if (rng.theta < 1) return SDR_E_INVALID;
  CanonView cv;
  int st = canonicalize(view, cv);
  if (st != SDR_OK) return st;
  if (cv.numel == 0) return SDR_OK;
  if (x == nullptr || y == nullptr) return SDR_E_INVALID;
  DropArgs A;
  memset(static_cast<void*>(&A), 0, sizeof(A));
  A.g = make_gen(rng);
  A.ix = make_indexer(cv);
  A.x = x;
  A.y = y;
  A.mask = mask;
  // keep-prob 1-p in float64 (rng.py:242), threshold ceil((1-p)*2^53).
  const double pk = 1.0 - p;
  const uint64_t T = static_cast<uint64_t>(ceil(pk * 9007199254740992.0));  // >= 1 as p < 1
  A.keep_le = (T >= (uint64_t{1} << 53)) ? ~uint64_t{0} : (T << 11) - 1;
  const double scale = 1.0 / (1.0 - p);
  A.scale64 = scale;
  A.scale32 = static_cast<float>(scale);
  A.scale16 = __half_as_ushort(__double2half(scale));
  bool fast = cv.istride == 1 && cv.inner % kDropCh == 0 && aligned16(x) && aligned16(y) &&
              (mask == nullptr || (reinterpret_cast<uintptr_t>(mask) & 7u) == 0);
  setup_chunks(cv, fast, A.nchunks, A.chunks_per_row, A.div_cpr, kDropCh);
  A.aligned = fast && chunks_aligned(cv, rng.theta, kDropCh);
  if (!fast && cv.istride == 1 && cv.inner >= kDropCh) {  // ragged rows: chunked Philox, per-element I/O
    A.ragged = 1;
    A.chunks_per_row = (static_cast<uint64_t>(cv.inner) + kDropCh - 1) / kDropCh;
    A.nchunks = static_cast<uint64_t>(cv.numel / cv.inner) * A.chunks_per_row;
    A.div_cpr = FastDiv64(A.chunks_per_row);
  }
  if (xt == SDR_F32 && yt == SDR_F32) return dispatch_drop_mask<SDR_F32, SDR_F32>(mt, A, fast, s);
  if (xt == SDR_F64 && yt == SDR_F64) return dispatch_drop_mask<SDR_F64, SDR_F64>(mt, A, fast, s);
  if (xt == SDR_BF16 && yt == SDR_BF16) return dispatch_drop_mask<SDR_BF16, SDR_BF16>(mt, A, fast, s);
  if (xt == SDR_BF16 && yt == SDR_F32) return dispatch_drop_mask<SDR_BF16, SDR_F32>(mt, A, fast, s);
  if (xt == SDR_F16 && yt == SDR_F16) return dispatch_drop_mask<SDR_F16, SDR_F16>(mt, A, fast, s);
  return SDR_E_DTYPE;
}

}  // namespace sdr
