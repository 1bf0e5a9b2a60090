// sdr_core.cuh -- shared device/host pieces of the sm_100a distributed RNG.
//
// Philox4x32-10 (reference: /root/reference/pkg/src/spmdsim/rng.py:34-59),
// the counter/key layout of _blocks_for (rng.py:76-82), fast 64-bit division
// for the tau/beta virtualisation (rng.py:198-201) and the canonical window
// ("CanonView") every Shard/Replicate/InterleavedShard window of a row-major
// tensor collapses to (placement.py:202-257).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "../../include/sdrng.h"

#define SDR_HD __host__ __device__ __forceinline__

namespace sdr {

constexpr uint32_t kM0 = 0xD2511F53u;  // rng.py:26
constexpr uint32_t kM1 = 0xCD9E8D57u;  // rng.py:27
constexpr uint32_t kW0 = 0x9E3779B9u;  // rng.py:28
constexpr uint32_t kW1 = 0xBB67AE85u;  // rng.py:29

// Elements per thread-chunk: one 16-byte bf16 vector, two f32 vectors.
constexpr int kV = 8;
constexpr int kMaxCanon = 2 * SDR_MAX_NDIM;

SDR_HD uint32_t hi32(uint64_t x) { return static_cast<uint32_t>(x >> 32); }
SDR_HD uint32_t lo32(uint64_t x) { return static_cast<uint32_t>(x); }
SDR_HD uint64_t mul_wide(uint32_t a, uint32_t b) { return static_cast<uint64_t>(a) * b; }

// Round keys k0 + r*W0, k1 + r*W1 for r = 0..9 (rng.py:57-58), precomputed on
// the host so the kernels read them as constant-bank operands.
struct RoundKeys {
  uint32_t k0[10];
  uint32_t k1[10];
};

inline RoundKeys make_keys(uint64_t seed) {
  RoundKeys k;
  uint32_t a = static_cast<uint32_t>(seed), b = static_cast<uint32_t>(seed >> 32);
  for (int r = 0; r < 10; ++r) {
    k.k0[r] = a;
    k.k1[r] = b;
    a += kW0;
    b += kW1;
  }
  return k;
}

// One Philox round: products M0*x0, M1*x2 split hi/lo; (rng.py:47-56).
SDR_HD void philox_round(uint32_t& x0, uint32_t& x1, uint32_t& x2, uint32_t& x3, uint32_t k0,
                         uint32_t k1) {
  const uint64_t pa = mul_wide(x0, kM0);
  const uint64_t pb = mul_wide(x2, kM1);
  const uint32_t y0 = hi32(pb) ^ x1 ^ k0;
  const uint32_t y2 = hi32(pa) ^ x3 ^ k1;
  x1 = lo32(pb);
  x3 = lo32(pa);
  x0 = y0;
  x2 = y2;
}

// Full 10-round block on counter (beta_lo, beta_hi, tau_lo, tau_hi).
SDR_HD void philox10(uint64_t seed, uint64_t tau, uint64_t beta, uint32_t w[4]) {
  uint32_t x0 = lo32(beta), x1 = hi32(beta), x2 = lo32(tau), x3 = hi32(tau);
  uint32_t k0 = lo32(seed), k1 = hi32(seed);
  for (int r = 0; r < 10; ++r) {
    philox_round(x0, x1, x2, x3, k0, k1);
    k0 += kW0;
    k1 += kW1;
  }
  w[0] = x0;
  w[1] = x1;
  w[2] = x2;
  w[3] = x3;
}

// Unsigned 64-bit division by a launch-constant divisor (Granlund-Montgomery,
// round-up variant; exact for every 64-bit numerator).
struct FastDiv64 {
  uint64_t d;
  uint64_t m;
  uint32_t s;
  uint32_t pow2;

  FastDiv64() : d(1), m(0), s(0), pow2(1) {}
  explicit FastDiv64(uint64_t div) : d(div), m(0), s(0), pow2(0) {
    if ((div & (div - 1)) == 0) {
      pow2 = 1;
      s = 0;
      while ((uint64_t{1} << s) < div) ++s;
      return;
    }
    uint32_t l = 0;
    while (l < 64 && (uint64_t{1} << l) < div) ++l;  // l = ceil(log2 d), 2..63
    unsigned __int128 num = (static_cast<unsigned __int128>(1) << 64) *
                            ((static_cast<unsigned __int128>(1) << l) - div);
    m = static_cast<uint64_t>(num / div) + 1;
    s = l - 1;
  }
  __device__ __forceinline__ uint64_t div(uint64_t n) const {
    if (pow2) return n >> s;
    const uint64_t t = __umul64hi(m, n);
    return (t + ((n - t) >> 1)) >> s;
  }
  __device__ __forceinline__ void divmod(uint64_t n, uint64_t& q, uint64_t& r) const {
    q = div(n);
    r = n - q * d;
  }
};

// A window reduced to: `nd` outer dims (outermost first) x one inner run.
// Local element i (row-major) has global flat index
//   base + sum_k digit_k(row) * ostride[k] + col * istride,
// row = i / inner, col = i % inner.
struct CanonView {
  int32_t nd;
  int32_t pad_;
  int64_t osize[kMaxCanon];
  int64_t ostride[kMaxCanon];
  int64_t inner;
  int64_t istride;
  int64_t base;
  int64_t numel;
};

// Build the canonical view; returns SDR_OK or SDR_E_INVALID.
int canonicalize(const sdr_view& v, CanonView& cv);

// Device: global flat index of local element i (generic path).
struct ViewIndexer {
  CanonView cv;
  FastDiv64 div_inner;
  FastDiv64 div_o[kMaxCanon];

  __device__ __forceinline__ uint64_t global_of(uint64_t i) const {
    uint64_t row, col;
    div_inner.divmod(i, row, col);
    uint64_t j = static_cast<uint64_t>(cv.base) + col * static_cast<uint64_t>(cv.istride);
    for (int k = cv.nd - 1; k >= 0; --k) {
      uint64_t q, r;
      div_o[k].divmod(row, q, r);
      j += r * static_cast<uint64_t>(cv.ostride[k]);
      row = q;
    }
    return j;
  }
};

inline ViewIndexer make_indexer(const CanonView& cv) {
  ViewIndexer ix;
  ix.cv = cv;
  ix.div_inner = FastDiv64(static_cast<uint64_t>(cv.inner > 0 ? cv.inner : 1));
  for (int k = 0; k < kMaxCanon; ++k)
    ix.div_o[k] = FastDiv64(static_cast<uint64_t>(k < cv.nd && cv.osize[k] > 0 ? cv.osize[k] : 1));
  return ix;
}

// Element sizes of sdr_dtype codes.
inline int dtype_size(int dt) {
  switch (dt) {
    case SDR_F32: case SDR_I32: return 4;
    case SDR_F64: case SDR_I64: return 8;
    case SDR_BF16: case SDR_F16: return 2;
    case SDR_U8: case SDR_BOOL: return 1;
    default: return 0;
  }
}

// Thread-local error bookkeeping for sdr_last_cuda_error().
void set_cuda_error(cudaError_t e);
int check_launch();

}  // namespace sdr
