// rng_kernels.cu -- sm_100a kernels for the single-device-semantic RNG.
//
// Every element e of a window gets ONE Philox4x32-10 block on counter
//   (beta_lo, beta_hi, tau_lo, tau_hi),  tau = j mod THETA, beta = j div THETA + offset,
// j = its global row-major flat index (rng.py:185-205).
// Values therefore depend only on (seed, offset, THETA, j): any rank produces
// exactly its slice of the unsharded tensor with no communication.
//
// Layout of the work: a thread owns chunks of kV = 8 consecutive local elements
// (one 16 B bf16 vector / two 16 B f32 vectors), grid-stride over the window.
// Fast path (unit inner stride; inner run % 8 == 0 with 16 B aligned buffers,
// or ragged rows with per-element I/O): the chunk's 8 global indices are
// consecutive, so when they share beta the round-1 product M0*beta_lo and the
// round-2 product M1*y2 are computed once per chunk and the round-1 products
// M1*(tau+e) are formed by 64-bit adds; the last round's M0 product is dead
// (every distribution uses words 0-1 only) -- about 14 IMAD.WIDE per element
// instead of 20.  Dropout needs only w1 (rounds 9-10 trimmed further).
//
// Normal (rng.py:141-156) is a certified fast path over NumPy's own float64
// transcendentals: a ~2^-40 table + polynomial evaluation of r and c whose
// error is measured exhaustively at load, a rigorous bound, and the exact
// NumPy tables for the few elements the bound cannot certify.
// The SDR_* macros below are A/B knobs; their defaults are the measured best.
#include <quadmath.h>
#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <type_traits>
#include <vector>

#include "rng_common.cuh"
#include "dist_transforms.cuh"

namespace sdr {

// Incremental chunk walk of a grid-stride loop over a view with at most one
// outer dim (nd <= 1): after one division for the first chunk, each step of
// S = gridDim*blockDim chunks adds dj to the global index and dcq to the
// column, with one conditional wrap to the next row.  Set per launch
// (set_walk) because S depends on the grid.
struct ChunkWalk {
  uint64_t dj, dcq, wrap;
  uint32_t on;  // nd <= 1
};

inline void set_walk(ChunkWalk& w, const CanonView& cv, uint64_t cpr, uint64_t S, int ch) {
  w.on = cv.nd <= 1 && cpr > 0 && cv.inner % ch == 0;  // (ragged rows take fill_chunk_ragged)
  if (!w.on) return;
  const uint64_t os0 = cv.nd == 1 ? static_cast<uint64_t>(cv.ostride[0]) : cpr * ch;
  w.dcq = S % cpr;
  w.dj = (S / cpr) * os0 + w.dcq * ch;
  w.wrap = os0 - cpr * ch;
}

// First chunk of this thread: global index and column (one division).
__device__ __forceinline__ uint64_t walk_start(const ViewIndexer& ix, const FastDiv64& div_cpr,
                                               uint64_t q, int ch, uint64_t& cq) {
  uint64_t row;
  div_cpr.divmod(q, row, cq);
  uint64_t j = static_cast<uint64_t>(ix.cv.base) + cq * ch;
  if (ix.cv.nd == 1) j += row * static_cast<uint64_t>(ix.cv.ostride[0]);
  return j;
}

__device__ __forceinline__ void walk_next(const ChunkWalk& w, uint64_t cpr, uint64_t& j, uint64_t& cq) {
  cq += w.dcq;
  j += w.dj;
  if (cq >= cpr) {
    cq -= cpr;
    j += w.wrap;
  }
}

// ---------------------------------------------------------------------------
// Fill kernels.
// ---------------------------------------------------------------------------
struct __align__(16) FillArgs {
  Gen g;
  DistP d;
  ViewIndexer ix;
  void* out;
  // Fast-path chunk walk: chunk q covers local [8q, 8q+8) inside one row.
  uint32_t aligned;  // THETA pow2 >= 8 and chunk starts 8-aligned (no straddle)
  uint32_t ragged;   // inner extent not a multiple of kV: per-element stores (fill_chunk_ragged)
  uint64_t nchunks;
  uint64_t chunks_per_row;
  FastDiv64 div_cpr;
  ChunkWalk walk;
};

// Global flat index of the first element of chunk q (fast path).
__device__ __forceinline__ uint64_t chunk_base(const FillArgs& A, uint64_t q) {
  if (A.ix.cv.nd == 0) return static_cast<uint64_t>(A.ix.cv.base) + q * kV;  // one contiguous run
  return outer_base(A.ix, A.div_cpr, q, kV);
}

template <int DIST, int DT, bool ALIGNED>
__device__ __forceinline__ void fill_chunk_at(const FillArgs& A, const NormalLut* L, uint64_t q,
                                              uint64_t j0);

// bfloat16 normal fills resolve uncertified elements through the per-warp
// queue (dist_transforms.cuh, MissQ); the kernels init it and flush it.
template <int DIST, int DT>
constexpr bool uses_missq() {
  return SDR_MISSQ && DIST == SDR_NORMAL && half_dt<DT>() && SDR_NORMAL_BF16_F32 && SDR_NSPLIT == 1;
}
static_assert(fill_threads<SDR_NORMAL, SDR_BF16>() <= 256, "MissQ (dist_transforms.cuh) holds 8 warps' queues");

template <int DIST, int DT, bool ALIGNED>
__device__ __forceinline__ void fill_chunk(const FillArgs& A, const NormalLut* L, uint64_t q) {
  fill_chunk_at<DIST, DT, ALIGNED>(A, L, q, chunk_base(A, q));
}

// Values of the kV elements with global indices j0 .. j0+kV-1.
template <int DIST, int DT>
__device__ __forceinline__ void values_from_words(const FillArgs& A, const NormalLut* L,
                                                  const uint32_t (&w0)[kV], const uint32_t (&w1)[kV],
                                                  typename St<DT>::T (&v)[kV]);

template <bool ALIGNED>
__device__ __forceinline__ void fill_words(const FillArgs& A, uint64_t j0, uint32_t (&w0)[kV],
                                           uint32_t (&w1)[kV]) {
  if constexpr (ALIGNED) chunk_words_aligned<kV>(A.g, j0, w0, w1);
  else chunk_words<kV>(A.g, j0, w0, w1);
}

// Transform of elements E0 .. E0+3 of a chunk from their words (the half-chunk
// pipeline of k_fill_fast).
template <int DT, int E0>
__device__ __forceinline__ void normal_half(const FillArgs& A, const NormalLut* L, const uint32_t (&w0)[4],
                                            const uint32_t (&w1)[4], typename St<DT>::T (&v)[kV]) {
  if constexpr (uses_lut2<SDR_NORMAL, DT>())
    normal_chunk2<DT, 4>(A.d, reinterpret_cast<const NormalLut2*>(L), w0, w1, v + E0);
  else
    normal_chunk_bf16<DT, 4>(A.d, reinterpret_cast<const NormalLut32*>(L), w0, w1, v + E0);
}

// Normal values of a chunk in SDR_NSPLIT parts (Philox words of a part, then
// its transform) so the peak register set is one part's, not the chunk's.
template <int DT, int NE, int E0>
__device__ __forceinline__ void normal_part(const FillArgs& A, const NormalLut* L, const ChunkHoist& H,
                                            typename St<DT>::T (&v)[kV]) {
  uint32_t w0[NE], w1[NE];
  words_part<NE, E0>(A.g.keys, H, w0, w1);
  if constexpr (uses_lut2<SDR_NORMAL, DT>())
    normal_chunk2<DT, NE>(A.d, reinterpret_cast<const NormalLut2*>(L), w0, w1, v + E0);
  else
    normal_chunk_bf16<DT, NE>(A.d, reinterpret_cast<const NormalLut32*>(L), w0, w1, v + E0);
  if constexpr (E0 + NE < kV) normal_part<DT, NE, E0 + NE>(A, L, H, v);
}

template <int DIST, int DT, bool ALIGNED>
__device__ __forceinline__ void chunk_values(const FillArgs& A, const NormalLut* L, uint64_t j0,
                                             typename St<DT>::T (&v)[kV]) {
  if constexpr (ALIGNED && SDR_NSPLIT > 1 && DIST == SDR_NORMAL &&
                (uses_lut2<DIST, DT>() || (half_dt<DT>() && SDR_NORMAL_BF16_F32))) {
    const ChunkHoist H = hoist_chunk(A.g, j0);
    normal_part<DT, kV / SDR_NSPLIT, 0>(A, L, H, v);
  } else {
    uint32_t w0[kV], w1[kV];
    fill_words<ALIGNED>(A, j0, w0, w1);
    values_from_words<DIST, DT>(A, L, w0, w1, v);
  }
}

template <int DIST, int DT>
__device__ __forceinline__ void values_from_words(const FillArgs& A, const NormalLut* L,
                                                  const uint32_t (&w0)[kV], const uint32_t (&w1)[kV],
                                                  typename St<DT>::T (&v)[kV]) {
  if constexpr (DIST == SDR_NORMAL && half_dt<DT>() && SDR_NORMAL_BF16_F32) {
    normal_chunk_bf16<DT, kV>(A.d, reinterpret_cast<const NormalLut32*>(L), w0, w1, v);
  } else if constexpr (uses_lut2<DIST, DT>()) {
    normal_chunk2<DT, kV>(A.d, reinterpret_cast<const NormalLut2*>(L), w0, w1, v);
  } else if constexpr (DIST == SDR_NORMAL && DT == SDR_F64) {
    normal_chunk_f64<kV>(A.d, L, w0, w1, v);
  } else if constexpr (DIST == SDR_NORMAL) {
    constexpr int NS = SDR_NORMAL_SPLIT;
#pragma unroll
    for (int h = 0; h < NS; ++h)
      normal_chunk<DT, kV / NS>(A.d, L, w0 + h * (kV / NS), w1 + h * (kV / NS), v + h * (kV / NS));
  } else {
#pragma unroll
    for (int e = 0; e < kV; ++e) v[e] = dist_value<DIST, DT>(A.d, L, w0[e], w1[e]);
  }
}

// Chunk q whose first element has global index j0.  bfloat16 normals queue
// their uncertified elements (MissQ) with this chunk's destination.
template <int DIST, int DT, bool ALIGNED>
__device__ __forceinline__ void fill_chunk_at(const FillArgs& A, const NormalLut* L, uint64_t q,
                                              uint64_t j0) {
  using T = typename St<DT>::T;
  T v[kV];
  T* dst = static_cast<T*>(A.out) + q * kV;
  if constexpr (uses_missq<DIST, DT>()) {
    uint32_t w0[kV], w1[kV];
    fill_words<ALIGNED>(A, j0, w0, w1);
    normal_chunk_bf16<DT, kV>(A.d, reinterpret_cast<const NormalLut32*>(L), w0, w1, v, dst);
  } else {
    chunk_values<DIST, DT, ALIGNED>(A, L, j0, v);
  }
  store_chunk(dst, v);
}

// Ragged rows (inner extent not a multiple of kV): chunk q = (row, cq) covers
// columns [kV cq, min(kV cq + kV, inner)) of its row; the Philox words are
// still computed kV at a time on consecutive global indices, the stores are
// per element (row starts are not 16 B aligned).
template <int DIST, int DT, bool ALIGNED>
__device__ __forceinline__ void fill_chunk_ragged(const FillArgs& A, const NormalLut* L, uint64_t q) {
  using T = typename St<DT>::T;
  const CanonView& cv = A.ix.cv;
  uint64_t row, cq;
  A.div_cpr.divmod(q, row, cq);
  uint64_t j0 = static_cast<uint64_t>(cv.base) + cq * kV, r = row;
  for (int k = cv.nd - 1; k >= 1; --k) {
    uint64_t qq, rem;
    A.ix.div_o[k].divmod(r, qq, rem);
    j0 += rem * static_cast<uint64_t>(cv.ostride[k]);
    r = qq;
  }
  if (cv.nd >= 1) j0 += r * static_cast<uint64_t>(cv.ostride[0]);
  const uint64_t inner = static_cast<uint64_t>(cv.inner);
  const uint64_t lq = row * inner + cq * kV;
  const int nvalid = static_cast<int>(min(static_cast<uint64_t>(kV), inner - cq * kV));
  T v[kV];
  T* out = static_cast<T*>(A.out) + lq;
  if constexpr (uses_missq<DIST, DT>()) {  // queue only the elements this row owns
    uint32_t w0[kV], w1[kV];
    fill_words<ALIGNED>(A, j0, w0, w1);
    normal_chunk_bf16<DT, kV>(A.d, reinterpret_cast<const NormalLut32*>(L), w0, w1, v, out, nvalid);
  } else {
    chunk_values<DIST, DT, ALIGNED>(A, L, j0, v);
  }
#pragma unroll
  for (int e = 0; e < kV; ++e)
    if (e < nvalid) out[e] = v[e];
}

template <int DIST, int DT>
__device__ __forceinline__ void fill_elem(const FillArgs& A, const NormalLut* L, uint64_t i) {
  using T = typename St<DT>::T;
  if constexpr (tablefree<DIST, DT>()) L = A.d.nm.lut;  // nothing staged: the float64 tables through L1
  uint32_t w0, w1;
  elem_words(A.g, A.ix.global_of(i), w0, w1);
  static_cast<T*>(A.out)[i] = dist_value<DIST, DT>(A.d, L, w0, w1);
}

template <int DIST, int DT, bool ALIGNED>
__global__ void __launch_bounds__(fill_threads<DIST, DT>(), fill_minb<DIST, DT>())
    k_fill_fast(const __grid_constant__ FillArgs A) {
#if SDR_PDL
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
  const NormalLut* L = nullptr;
  uint32_t bar = 0;  // Normal: tables arriving by TMA (waited on before first use)
  if constexpr (tablefree<DIST, DT>()) {
    // bfloat16 on the MUFU functions: nothing to stage
  } else if constexpr (uses_lut2<DIST, DT>()) {
    extern __shared__ __align__(16) unsigned char s_dyn[];  // sizeof(NormalLut2), set at launch
    NormalLut2* s_lut2 = reinterpret_cast<NormalLut2*>(s_dyn);
    bar = stage_lut_begin(s_lut2, A.d.nm.lut2);
    L = reinterpret_cast<const NormalLut*>(s_lut2);
  } else if constexpr (DIST == SDR_NORMAL && half_dt<DT>() && SDR_NORMAL_BF16_F32) {
    extern __shared__ __align__(16) unsigned char s_dyn[];  // sizeof(NormalLut32), set at launch
    NormalLut32* s_lut32 = reinterpret_cast<NormalLut32*>(s_dyn);
    bar = stage_lut_begin(s_lut32, A.d.nm.lut32);
    L = reinterpret_cast<const NormalLut*>(s_lut32);
  } else if constexpr (DIST == SDR_NORMAL) {
    __shared__ __align__(16) NormalLut s_lut;
    bar = stage_lut_begin(&s_lut, A.d.nm.lut);
    L = &s_lut;
  }
#if SDR_PDL
  // previous grid's memory visible before any store (the constant tables may
  // already be in flight: they are never written by a kernel)
  asm volatile("griddepcontrol.wait;" ::: "memory");
#endif
  if constexpr (uses_missq<DIST, DT>()) missq_init();
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  uint64_t q = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (A.walk.on) {
    uint64_t cq;
    uint64_t j = walk_start(A.ix, A.div_cpr, q, kV, cq);
    if constexpr (DIST == SDR_NORMAL && SDR_FILL_PIPE == 2 && ALIGNED &&
                  (uses_lut2<DIST, DT>() || (half_dt<DT>() && SDR_NORMAL_BF16_F32))) {
      // Half-chunk software pipeline: every step computes the Philox words of
      // the NEXT half chunk (4 elements; pure arithmetic, computed past the end
      // too and discarded) in the same basic block as the transform of the
      // current half, so the fma-heavy IMAD.WIDE stream and the transform's
      // ALU / FP32 / shared / XU work interleave inside each warp.
      using T = typename St<DT>::T;
      ChunkHoist H = hoist_chunk(A.g, j);
      uint32_t a0[4], a1[4], b0[4], b1[4];
      words_part<4, 0>(A.g.keys, H, a0, a1);
      if constexpr (stages_lut<DIST, DT>()) stage_lut_wait(bar);
      for (; q < A.nchunks; q += stride) {
        T v[kV];
        words_part<4, 4>(A.g.keys, H, b0, b1);
        normal_half<DT, 0>(A, L, a0, a1, v);
        uint64_t jn = j, cqn = cq;
        walk_next(A.walk, A.chunks_per_row, jn, cqn);
        H = hoist_chunk(A.g, jn);
        words_part<4, 0>(A.g.keys, H, a0, a1);
        normal_half<DT, 4>(A, L, b0, b1, v);
        store_chunk(static_cast<T*>(A.out) + q * kV, v);
        j = jn;
        cq = cqn;
      }
    } else if constexpr (DIST == SDR_NORMAL && SDR_FILL_PIPE == 1) {
      // Software pipeline: the Philox words of the thread's next chunk are
      // computed (unconditionally: pure arithmetic, discarded past the end)
      // in the same basic block as the transform of the current chunk, so the
      // fma-heavy IMAD.WIDE stream interleaves with the transform's ALU /
      // shared / XU work instead of alternating phases.
      using T = typename St<DT>::T;
      uint32_t w0[kV], w1[kV];
      fill_words<ALIGNED>(A, j, w0, w1);
      if constexpr (stages_lut<DIST, DT>()) stage_lut_wait(bar);
      for (; q < A.nchunks; q += stride) {
        uint64_t jn = j, cqn = cq;
        walk_next(A.walk, A.chunks_per_row, jn, cqn);
        uint32_t n0[kV], n1[kV];
        fill_words<ALIGNED>(A, jn, n0, n1);
        T v[kV];
        values_from_words<DIST, DT>(A, L, w0, w1, v);
        store_chunk(static_cast<T*>(A.out) + q * kV, v);
#pragma unroll
        for (int e = 0; e < kV; ++e) {
          w0[e] = n0[e];
          w1[e] = n1[e];
        }
        j = jn;
        cq = cqn;
      }
    } else if constexpr (DIST == SDR_NORMAL) {
      // first chunk peeled: its Philox words overlap the table transfer
      if (q < A.nchunks) {
        using T = typename St<DT>::T;
        uint32_t w0[kV], w1[kV];
        fill_words<ALIGNED>(A, j, w0, w1);
        if constexpr (stages_lut<DIST, DT>()) stage_lut_wait(bar);
        T v[kV];
        T* dst = static_cast<T*>(A.out) + q * kV;
        if constexpr (uses_missq<DIST, DT>())
          normal_chunk_bf16<DT, kV>(A.d, reinterpret_cast<const NormalLut32*>(L), w0, w1, v, dst);
        else
          values_from_words<DIST, DT>(A, L, w0, w1, v);
        store_chunk(dst, v);
        walk_next(A.walk, A.chunks_per_row, j, cq);
        q += stride;
      } else if constexpr (stages_lut<DIST, DT>()) {
        stage_lut_wait(bar);
      }
    }
    if constexpr (uses_missq<DIST, DT>()) {
      // warp-uniform trip count, so the converged warp can resolve its miss
      // queue every few chunks (no overflow into the inline path on large
      // fills, no flush burst at the end of the kernel)
      const unsigned my_iters =
          q < A.nchunks ? static_cast<unsigned>((A.nchunks - q + stride - 1) / stride) : 0u;
      const unsigned iters = __reduce_max_sync(0xffffffffu, my_iters);
      // up to 24 chunks per thread the queue (256) cannot fill at ~1% misses:
      // the plain loop (measured 6% faster there) and one flush at the end
      if (iters <= 24u) {
        for (; q < A.nchunks; q += stride) {
          fill_chunk_at<DIST, DT, ALIGNED>(A, L, q, j);
          walk_next(A.walk, A.chunks_per_row, j, cq);
        }
      } else for (unsigned it = 0; it < iters; ++it) {
        if (q < A.nchunks) {
          fill_chunk_at<DIST, DT, ALIGNED>(A, L, q, j);
          walk_next(A.walk, A.chunks_per_row, j, cq);
        }
        q += stride;
        if ((it & 7u) == 7u) {
          __syncwarp();
          if (missq()->n >= 64u) missq_flush<DT>(A.d);  // n is the warp's own: a uniform branch
        }
      }
    } else {
      for (; q < A.nchunks; q += stride) {
        fill_chunk_at<DIST, DT, ALIGNED>(A, L, q, j);
        walk_next(A.walk, A.chunks_per_row, j, cq);
      }
    }
  } else if (A.ragged) {
    if constexpr (stages_lut<DIST, DT>()) stage_lut_wait(bar);
    for (; q < A.nchunks; q += stride) fill_chunk_ragged<DIST, DT, ALIGNED>(A, L, q);
  } else {
    if constexpr (stages_lut<DIST, DT>()) stage_lut_wait(bar);
    for (; q < A.nchunks; q += stride) fill_chunk<DIST, DT, ALIGNED>(A, L, q);
  }
  if constexpr (uses_missq<DIST, DT>()) missq_flush<DT>(A.d);  // every thread gets here: the warp is converged
}

template <int DIST, int DT>
__global__ void __launch_bounds__(256) k_fill_generic(const __grid_constant__ FillArgs A) {
  const NormalLut* L = nullptr;
  if constexpr (DIST == SDR_NORMAL) {
    __shared__ __align__(16) NormalLut s_lut;
    stage_lut(&s_lut, A.d.nm.lut);
    L = &s_lut;
  }
  const uint64_t n = static_cast<uint64_t>(A.ix.cv.numel);
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += stride)
    fill_elem<DIST, DT>(A, L, i);
}

// Multi-tensor fill (K3): the members of one (distribution, dtype) group are
// cut into tiles of kTileElems elements; CTAs walk the global tile list, stage
// the member's descriptor in shared memory once per tile and fill it.  One
// launch initialises every parameter of a model (model.py:121-132).
#ifndef SDR_TILE_ELEMS
#define SDR_TILE_ELEMS 131072  // elements per tile of the batched fill (measured: 16K..256K, 128K best overall)
#endif
constexpr uint64_t kTileElems = SDR_TILE_ELEMS;

template <int DIST, int DT>
__global__ void __launch_bounds__(fill_threads<DIST, DT>(), fill_minb<DIST, DT>())
    k_fill_batch(const FillArgs* __restrict__ descs, const uint64_t* __restrict__ tile_prefix, int n,
                 uint64_t ntiles, unsigned long long* __restrict__ next_tile) {
  __shared__ __align__(16) unsigned char smem[sizeof(FillArgs)];
  FillArgs& A = *reinterpret_cast<FillArgs*>(smem);
  const NormalLut* L = nullptr;
  if constexpr (tablefree<DIST, DT>()) {
    // bfloat16 on the MUFU functions: nothing to stage
  } else if constexpr (uses_lut2<DIST, DT>()) {
    extern __shared__ __align__(16) unsigned char s_dyn[];  // sizeof(NormalLut2), set at launch
    NormalLut2* s_lut2 = reinterpret_cast<NormalLut2*>(s_dyn);
    stage_lut(s_lut2, descs[0].d.nm.lut2);
    L = reinterpret_cast<const NormalLut*>(s_lut2);
  } else if constexpr (DIST == SDR_NORMAL && half_dt<DT>() && SDR_NORMAL_BF16_F32) {
    extern __shared__ __align__(16) unsigned char s_dyn[];  // sizeof(NormalLut32), set at launch
    NormalLut32* s_lut32 = reinterpret_cast<NormalLut32*>(s_dyn);
    stage_lut(s_lut32, descs[0].d.nm.lut32);
    L = reinterpret_cast<const NormalLut*>(s_lut32);
  } else if constexpr (DIST == SDR_NORMAL) {
    __shared__ __align__(16) NormalLut s_lut;
    stage_lut(&s_lut, descs[0].d.nm.lut);
    L = &s_lut;
  }
  if constexpr (uses_missq<DIST, DT>()) missq_init();
  // Persistent CTAs take tiles from a launch-wide counter (zeroed by the
  // descriptor upload): members differ in size and their last tiles are
  // partial, so a fixed tile-to-CTA map left the grid unbalanced (measured:
  // 27.9 ms for one wave with a static map, 26.7-26.9 ms with 4-5x
  // oversubscription; the counter balances without oversubscribing).
  __shared__ unsigned long long s_tile;
  for (;;) {
    __syncthreads();  // previous tile done with A and s_tile
    if (threadIdx.x == 0) s_tile = atomicAdd(next_tile, 1ull);
    __syncthreads();
    const uint64_t t = s_tile;
    if (t >= ntiles) break;
    // member f: last index with tile_prefix[f] <= t (uniform across the CTA)
    int lo = 0, hi = n - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (tile_prefix[mid] <= t) lo = mid;
      else hi = mid - 1;
    }
    {
      const uint4* src = reinterpret_cast<const uint4*>(descs + lo);
      uint4* dst = reinterpret_cast<uint4*>(smem);
      for (int i = threadIdx.x; i < static_cast<int>(sizeof(FillArgs) / 16); i += blockDim.x)
        dst[i] = src[i];
    }
    __syncthreads();
    const uint64_t lt = t - tile_prefix[lo];
    if (A.nchunks > 0) {
      const uint64_t q0 = lt * (kTileElems / kV);
      uint64_t q1 = q0 + kTileElems / kV;
      if (q1 > A.nchunks) q1 = A.nchunks;
      if (A.aligned) {
        for (uint64_t q = q0 + threadIdx.x; q < q1; q += blockDim.x) fill_chunk<DIST, DT, true>(A, L, q);
      } else {
        for (uint64_t q = q0 + threadIdx.x; q < q1; q += blockDim.x) fill_chunk<DIST, DT, false>(A, L, q);
      }
    } else {
      const uint64_t i0 = lt * kTileElems;
      uint64_t i1 = i0 + kTileElems;
      const uint64_t numel = static_cast<uint64_t>(A.ix.cv.numel);
      if (i1 > numel) i1 = numel;
      for (uint64_t i = i0 + threadIdx.x; i < i1; i += blockDim.x) fill_elem<DIST, DT>(A, L, i);
    }
    // this tile's queued elements, with this member's parameters (converged:
    // the tile loops are done; A is replaced only after the next barrier)
    if constexpr (uses_missq<DIST, DT>()) missq_flush<DT>(A.d);
  }
}

// Raw Philox words for (tau, beta) arrays (KAT / debug entry).
__global__ void k_philox_blocks(const uint64_t* tau, const uint64_t* beta, int64_t n,
                                const __grid_constant__ RoundKeys K, uint32_t* words) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint32_t x0 = lo32(beta[i]), x1 = hi32(beta[i]), x2 = lo32(tau[i]), x3 = hi32(tau[i]);
#pragma unroll
  for (int r = 0; r < 10; ++r) philox_round(x0, x1, x2, x3, K.k0[r], K.k1[r]);
  words[4 * i + 0] = x0;
  words[4 * i + 1] = x1;
  words[4 * i + 2] = x2;
  words[4 * i + 3] = x3;
}

// Distribution.transform (rng.py:104-182): words -> values, elementwise, with
// the same device transform the fill kernels use.
template <int DIST, int DT>
__global__ void __launch_bounds__(256) k_transform(const uint32_t* __restrict__ w0,
                                                   const uint32_t* __restrict__ w1, int64_t n,
                                                   const __grid_constant__ DistP P, void* out) {
  const NormalLut* L = nullptr;
  if constexpr (DIST == SDR_NORMAL) {
    __shared__ __align__(16) NormalLut s_lut;
    stage_lut(&s_lut, P.nm.lut);
    L = &s_lut;
  }
  using T = typename St<DT>::T;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
    static_cast<T*>(out)[i] = dist_value<DIST, DT>(P, L, __ldg(w0 + i), __ldg(w1 + i));
}

// Exhaustive calibration of the Normal fast path against the NumPy tables:
// max relative error of r_fast (k >= 1; k = 0 must give r <= 2^-490), max
// absolute error of c_fast, and the same for the float32 functions.
__global__ void k_normal_calibrate(const double* ltab, const double* ctab, const NormalLut* lut,
                                   const NormalLut32* lut32, const NormalLut2* lut2,
                                   unsigned long long* max_r_bits, unsigned long long* max_c_bits) {
  __shared__ __align__(16) NormalLut s_lut;
  stage_lut(&s_lut, lut);  // the float32 tables are read from global memory here
  const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= (1u << 24)) return;
  const double inf = __longlong_as_double(0x7FF0000000000000ll);
  const double rg = r_fast(k << 8, &s_lut, -0.5, 1.5), rn = __dsqrt_rn(-2.0 * ltab[k]);  // NumPy's r
  double er;
  if (k == 0) er = (rn == 0.0 && rg >= 0.0 && rg <= 0x1p-490) ? 0.0 : inf;
  else er = (rg > 0.0 && rn > 0.0) ? fabs(rg - rn) / rg : inf;
  const double ec = fabs(c_fast(k << 8, &s_lut) - ctab[k]);
  const double r32 = r32_fast(k << 8, lut32);
  double er32;
  if (k == 0) er32 = (r32 >= 0.0 && r32 <= 0x1p-49) ? 0.0 : inf;
  else er32 = (r32 > 0.0 && rn > 0.0) ? fabs(r32 - rn) / r32 : inf;
  const double ec32 = fabs(static_cast<double>(c32_fast(k << 8, lut32)) - ctab[k]);  // absolute
  // NormalLut2 functions (tables read from global memory here)
  const double r2 = r_fast2(k << 8, lut2, -0.5, 1.5);
  double er2;
  if (k == 0) er2 = (r2 >= 0.0 && r2 <= 0x1p-490) ? 0.0 : inf;
  else er2 = (r2 > 0.0 && rn > 0.0) ? fabs(r2 - rn) / r2 : inf;
  const double ec2 = fabs(c_fast2(k << 8, lut2) - ctab[k]);
  unsigned long long b[6] = {static_cast<unsigned long long>(__double_as_longlong(er)),
                             static_cast<unsigned long long>(__double_as_longlong(ec)),
                             static_cast<unsigned long long>(__double_as_longlong(er32)),
                             static_cast<unsigned long long>(__double_as_longlong(ec32)),
                             static_cast<unsigned long long>(__double_as_longlong(er2)),
                             static_cast<unsigned long long>(__double_as_longlong(ec2))};
  // Non-negative doubles order like their bit patterns (NaN above inf); reduce per warp first.
#pragma unroll
  for (int i = 0; i < 6; ++i) {
    for (int o = 16; o > 0; o >>= 1) b[i] = max(b[i], __shfl_xor_sync(0xffffffffu, b[i], o));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMax(max_r_bits, b[0]);
    atomicMax(max_c_bits, b[1]);
    atomicMax(max_r_bits + 2, b[2]);
    atomicMax(max_c_bits + 2, b[3]);
    atomicMax(max_r_bits + 4, b[4]);
    atomicMax(max_c_bits + 4, b[5]);
  }
}

// Calibration of r32_mufu (bfloat16 path) over k in [1, 2^24): out[0] = Er =
// max |r - r_np| / r where r >= 1, out[1] = Ei = max |r - r_np| / h where r < 1,
// so |r - r_np| <= Er r + Ei h everywhere.  k = 0 is never certified (h = 2^60).
__global__ void k_normal_calibrate_mufu(const double* ltab, const double* ctab, unsigned long long* out) {
  const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= (1u << 24)) return;
  const double inf = __longlong_as_double(0x7FF0000000000000ll);
  float h;
  const double r = r32_mufu(k << 8, h), rn = __dsqrt_rn(-2.0 * ltab[k]);
  double er = 0.0, ei = 0.0;
  if (k > 0) {
    const double e = fabs(r - rn);
    if (!(r > 0.0) || !(h > 0.0f) || isinf(r) || isinf(h)) er = ei = inf;
    else if (r >= 1.0) er = e / r;
    else ei = e / static_cast<double>(h);
  }
  const double ec = fabs(static_cast<double>(c32_mufu(k << 8)) - ctab[k]);  // MUFU cosine, absolute
  unsigned long long b[3] = {static_cast<unsigned long long>(__double_as_longlong(er)),
                             static_cast<unsigned long long>(__double_as_longlong(ei)),
                             static_cast<unsigned long long>(__double_as_longlong(isnan(ec) ? inf : ec))};
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    for (int o = 16; o > 0; o >>= 1) b[i] = max(b[i], __shfl_xor_sync(0xffffffffu, b[i], o));
    if ((threadIdx.x & 31) == 0) atomicMax(out + i, b[i]);
  }
}

// ExactMirror construction: thread t owns table points 16t .. 16t+15 (one code
// word per function); exceptions are appended to unsorted lists.
__device__ __forceinline__ uint32_t mirror_code(double np, double cu) {
  const long long a = __double_as_longlong(np), b = __double_as_longlong(cu);
  if ((a ^ b) < 0) return a == b ? 0u : 3u;  // sign differs (only near a zero crossing)
  const long long d = a - b;
  return d == 0 ? 0u : d == 1 ? 1u : d == -1 ? 2u : 3u;
}
__global__ void k_mirror_codes(const double* __restrict__ ltab, const double* __restrict__ ctab,
                               uint32_t* code_l, uint32_t* code_c, uint32_t* xk_l, double* xv_l,
                               uint32_t* xk_c, double* xv_c, unsigned int* counts, unsigned int cap) {
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (1u << 20)) return;
  uint32_t wl = 0, wc = 0;
  for (uint32_t i = 0; i < 16; ++i) {
    const uint32_t k = 16u * t + i;
    const double cl = log1p(-static_cast<double>(k) * 0x1p-24);
    const double cc = cos(__dmul_rn(6.283185307179586, static_cast<double>(k) * 0x1p-24));
    const uint32_t a = mirror_code(ltab[k], cl), b = mirror_code(ctab[k], cc);
    wl |= a << (2 * i);
    wc |= b << (2 * i);
    if (a == 3u) {
      const unsigned int n = atomicAdd(counts, 1u);
      if (n < cap) {
        xk_l[n] = k;
        xv_l[n] = ltab[k];
      }
    }
    if (b == 3u) {
      const unsigned int n = atomicAdd(counts + 1, 1u);
      if (n < cap) {
        xk_c[n] = k;
        xv_c[n] = ctab[k];
      }
    }
  }
  code_l[t] = wl;
  code_c[t] = wc;
}

// Every table point through the compact mirror against NumPy's values, bit for bit.
__global__ void k_mirror_verify(const ExactMirror M, const double* __restrict__ ltab,
                                const double* __restrict__ ctab, unsigned long long* bad) {
  const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= (1u << 24)) return;
  const bool ok = __double_as_longlong(mirror_r(M, k)) == __double_as_longlong(__dsqrt_rn(-2.0 * ltab[k])) &&
                  __double_as_longlong(mirror_c(M, k)) == __double_as_longlong(ctab[k]);
  if (!ok) atomicAdd(bad, 1ull);
}

// float64 Normal corrections (normal_chunk_f64): for every table point k the
// difference between the bits of NumPy's r[k] / c[k] (the verified mirror, or
// the full tables) and of the fast functions, kDeltaEsc when it does not fit
// in 16 bits.  stats[0..1]: escapes of r / c, stats[2..3]: max |difference|
// stored.
__global__ void k_normal_deltas(const ExactMirror M, const double* __restrict__ rtab,
                                const double* __restrict__ ctab, const NormalLut* lut, DeltaR* dr,
                                int16_t* dc, unsigned long long* stats) {
  __shared__ __align__(16) NormalLut s_lut;
  stage_lut(&s_lut, lut);  // as the fill kernels read it
  const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= (1u << 24)) return;
  const double rn = rtab != nullptr ? rtab[k] : mirror_r(M, k);
  const double cn = ctab != nullptr ? ctab[k] : mirror_c(M, k);
  const long long a = __double_as_longlong(rn) - __double_as_longlong(r_unit(k << 8, &s_lut));
  const long long b = __double_as_longlong(cn) - __double_as_longlong(c_fast(k << 8, &s_lut));
  const bool fa = a > kDeltaEscR && a <= kDeltaMaxR, fb = dc == nullptr || (b > kDeltaEsc && b < 32768);
  dr[k] = static_cast<DeltaR>(fa ? a : kDeltaEscR);
  if (dc != nullptr) dc[k] = static_cast<int16_t>(fb ? b : kDeltaEsc);
  const unsigned ea = __popc(__ballot_sync(0xffffffffu, !fa)), eb = __popc(__ballot_sync(0xffffffffu, !fb));
  unsigned long long ma = fa ? static_cast<unsigned long long>(a < 0 ? -a : a) : 0ull;
  unsigned long long mb = fb && dc != nullptr ? static_cast<unsigned long long>(b < 0 ? -b : b) : 0ull;
  for (int o = 16; o > 0; o >>= 1) {
    ma = max(ma, __shfl_xor_sync(0xffffffffu, ma, o));
    mb = max(mb, __shfl_xor_sync(0xffffffffu, mb, o));
  }
  if ((threadIdx.x & 31) == 0) {
    if (ea) atomicAdd(stats, static_cast<unsigned long long>(ea));
    if (eb) atomicAdd(stats + 1, static_cast<unsigned long long>(eb));
    atomicMax(stats + 2, ma);
    atomicMax(stats + 3, mb);
  }
}

// c_cr against NumPy's c[k] on every table point: dc8[k] = bits(c_np) -
// bits(c_cr) for the flagged points (-128 when it does not fit), 0 elsewhere.
// stats: [0] flagged, [1] escapes, [2] unflagged mismatches (must be 0 for
// c_cr to be used), [3] max |difference| stored.
__global__ void k_normal_cos_cr(const ExactMirror M, const double* __restrict__ ctab, const NormalMirror NM,
                                int8_t* dc8, unsigned long long* stats) {
  const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= (1u << 24)) return;
  const double cn = ctab != nullptr ? ctab[k] : mirror_c(M, k);
  bool flag;
  const double c = c_cr(k << 8, NM.cdd, flag);
  const long long d = __double_as_longlong(cn) - __double_as_longlong(c);
  const bool fits = d > -128 && d < 128;
  dc8[k] = static_cast<int8_t>(flag ? (fits ? d : -128) : 0);
  const unsigned nf = __popc(__ballot_sync(0xffffffffu, flag));
  const unsigned ne = __popc(__ballot_sync(0xffffffffu, flag && !fits));
  const unsigned nb = __popc(__ballot_sync(0xffffffffu, !flag && d != 0));
  unsigned long long m = flag && fits ? static_cast<unsigned long long>(d < 0 ? -d : d) : 0ull;
  for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) {
    if (nf) atomicAdd(stats, static_cast<unsigned long long>(nf));
    if (ne) atomicAdd(stats + 1, static_cast<unsigned long long>(ne));
    if (nb) atomicAdd(stats + 2, static_cast<unsigned long long>(nb));
    atomicMax(stats + 3, m);
  }
}

// Full-table fallback: r[k] = sqrt(-2 L[k]) in place.
__global__ void k_r_from_l(double* t) {
  const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < (1u << 24)) t[k] = __dsqrt_rn(-2.0 * t[k]);
}

// ---------------------------------------------------------------------------
// Host side.
// ---------------------------------------------------------------------------
static thread_local char g_cuda_err[256] = "";

void set_cuda_error(cudaError_t e) {
  snprintf(g_cuda_err, sizeof(g_cuda_err), "%s: %s", cudaGetErrorName(e), cudaGetErrorString(e));
}

int check_launch() {
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_cuda_error(e);
    return SDR_E_CUDA;
  }
  return SDR_OK;
}

int canonicalize(const sdr_view& v, CanonView& cv) {
  if (v.ndim < 0 || v.ndim > SDR_MAX_NDIM) return SDR_E_INVALID;
  int64_t size[kMaxCanon], stride[kMaxCanon];
  int n = 0;
  int64_t pi = 1, base = 0, numel = 1;
  // Row-major global strides, innermost last.
  int64_t gstr[SDR_MAX_NDIM];
  for (int d = v.ndim - 1; d >= 0; --d) {
    if (v.global_shape[d] < 0) return SDR_E_INVALID;
    gstr[d] = pi;
    pi *= (v.global_shape[d] > 0 ? v.global_shape[d] : 1);
  }
  for (int d = 0; d < v.ndim; ++d) {
    const int64_t G = v.global_shape[d], s = v.local_start[d], len = v.local_len[d];
    const int64_t m = v.groups[d] > 0 ? v.groups[d] : 1;
    if (s < 0 || len < 0) return SDR_E_INVALID;
    numel *= len;
    if (m == 1) {
      if (len > 0 && s + len > G) return SDR_E_INVALID;
      base += s * gstr[d];
      size[n] = len;
      stride[n] = gstr[d];
      ++n;
    } else {
      if (len % m != 0) return SDR_E_INVALID;
      const int64_t per = len / m, gs = v.group_stride[d];
      if (per > 0 && (gs < per || s + (m - 1) * gs + per > G)) return SDR_E_INVALID;
      base += s * gstr[d];
      size[n] = m;
      stride[n] = gs * gstr[d];
      ++n;
      size[n] = per;
      stride[n] = gstr[d];
      ++n;
    }
  }
  cv = CanonView{};
  cv.numel = numel;
  cv.base = base;
  if (numel == 0) {
    cv.nd = 0;
    cv.inner = 1;
    cv.istride = 1;
    return SDR_OK;
  }
  // Drop size-1 dims, then merge (outer, inner) pairs that are contiguous.
  int64_t ms[kMaxCanon], mst[kMaxCanon];
  int k = 0;
  for (int i = 0; i < n; ++i) {
    if (size[i] == 1) continue;
    if (k > 0 && mst[k - 1] == size[i] * stride[i]) {
      ms[k - 1] *= size[i];
      mst[k - 1] = stride[i];
    } else {
      ms[k] = size[i];
      mst[k] = stride[i];
      ++k;
    }
  }
  if (k == 0) {
    cv.nd = 0;
    cv.inner = 1;
    cv.istride = 1;
    return SDR_OK;
  }
  cv.inner = ms[k - 1];
  cv.istride = mst[k - 1];
  cv.nd = k - 1;
  for (int i = 0; i < k - 1; ++i) {
    cv.osize[i] = ms[i];
    cv.ostride[i] = mst[i];
  }
  return SDR_OK;
}

// Per-device Normal mirror tables.
constexpr size_t kDeltaBytes = (sizeof(int16_t) + sizeof(DeltaR)) << 24;  // cmode 0: dc then dr
constexpr size_t kDeltaBytesCr = (sizeof(int8_t) + sizeof(DeltaR)) << 24;  // cmode 1: dr then dc8
struct NormalState {
  double* rtab = nullptr;  // full tables: only if the compact mirror failed verification
  double* ctab = nullptr;
  uint32_t* code = nullptr;  // 2 x 2^20 code words
  uint32_t* xk = nullptr;    // exception keys (l then c)
  double* xv = nullptr;      // exception values
  int nx_l = 0, nx_c = 0;
  uint64_t device_bytes = 0;  // mirror bytes resident on the device
  double build_ms = 0;
  NormalLut* lut = nullptr;
  NormalLut32* lut32 = nullptr;
  NormalLut2* lut2 = nullptr;
  unsigned long long* fallbacks = nullptr;
  double err_r = 0, err_c = 0, err_r32 = 0, err_c32 = 0, err_r2 = 0, err_c2 = 0;
  double err_rm = 0, err_im = 0, err_cm = 0;  // r32_mufu, c32_mufu (bfloat16 path)
  unsigned char* delta = nullptr;      // float64 corrections (layout by cmode, kDeltaBytes / kDeltaBytesCr), or null
  unsigned long long delta_stats[4] = {0, 0, 0, 0};  // escapes r / c, max |difference| r / c
  unsigned long long cr_stats[4] = {0, 0, 0, 0};     // c_cr: flagged, escapes, unflagged mismatches, max |d|
  CosDD* cdd = nullptr;                // c_cr's table (cmode 1)
  int cmode = 0;
  bool loaded = false;
};
static std::mutex g_nm_mu;

static double round_sig(long double x, int bits) {
  int e = 0;
  const long double m = frexpl(x, &e);  // x = m * 2^e, m in [0.5, 1)
  return static_cast<double>(ldexpl(nearbyintl(ldexpl(m, bits)), e - bits));
}

// c_cr's table: (cos, sin)(i pi/1024) for i in [0, 2048] as double-doubles
// from quad precision.
static void build_cos_dd(CosDD* T) {
  const __float128 Q = strtoflt128("3.14159265358979323846264338327950288419716939937510", nullptr) / 1024;
  for (int i = 0; i < kCosDD; ++i) {
    const __float128 c = cosq(Q * i), s = sinq(Q * i);
    T[i].ch = static_cast<double>(c);
    T[i].cl = static_cast<double>(c - static_cast<__float128>(T[i].ch));
    T[i].sh = static_cast<double>(s);
    T[i].sl = static_cast<double>(s - static_cast<__float128>(T[i].sh));
  }
  // c_cr's constant split of pi/1024 (kQ1 + kQ2 + kQ3) must match the quad value
  const __float128 r = Q - kQ1 - kQ2 - kQ3;
  if (fabsq(r) > Q * static_cast<__float128>(1e-32)) fprintf(stderr, "sdr: pi/1024 split is off by %g\n", static_cast<double>(r));
}

// Host construction of the fast-path tables (long double arithmetic).
static void build_normal_lut(NormalLut& L) {
  for (int j = 0; j < 512; ++j) {
    long double inv, mult;
    if (j == 0 || j == 511) {
      inv = 1.0L;
      mult = (j == 511) ? 0.5L : 1.0L;
    } else if (j < 256) {
      const long double mc = 1.0L + (j + 0.5L) / 512.0L;
      inv = round_sig(1.0L / mc, 20);
      mult = inv;
    } else {
      const long double mc = (1.0L + (j + 0.5L) / 512.0L) / 2.0L;
      inv = round_sig(1.0L / mc, 20);
      mult = inv / 2.0L;
    }
    L.logt[j].x = static_cast<double>(-2.0L * ldexpl(mult, -23));
    L.logt[j].y = (inv == 1.0L) ? 0.0 : static_cast<double>(2.0L * logl(inv));
  }
  L.logt[0].y = 0x1p-1000;
  const long double pi = 3.141592653589793238462643383279502884L;
  for (int i = 0; i < 2048; ++i) {
    const long double a = pi * i / 1024.0L;
    L.trig[i].x = static_cast<double>(cosl(a));
    L.trig[i].y = static_cast<double>(sinl(a));
  }
  // exact table points
  L.trig[0] = make_double2(1.0, 0.0);
  L.trig[512] = make_double2(0.0, 1.0);
  L.trig[1024] = make_double2(-1.0, 0.0);
  L.trig[1536] = make_double2(0.0, -1.0);
}

// float32 tables of the bfloat16 path: the float64 log table rounded (the
// logt.x entries are exact: 20-bit mult) and the two-level cosine table.
static void build_normal_lut32(const NormalLut& h, NormalLut32& L) {
  for (int j = 0; j < 512; ++j)
    L.logt[j] = make_float2(static_cast<float>(h.logt[j].x), static_cast<float>(h.logt[j].y));
  L.logt[0].y = 0x1p-100f;
  const long double pi = 3.141592653589793238462643383279502884L;
  for (int i = 0; i < 4096; ++i) {
    const long double a = 2.0L * pi * i / 4096.0L, b = 2.0L * pi * i / 16777216.0L;
    L.trig_hi[i] = make_float2(static_cast<float>(cosl(a)), static_cast<float>(sinl(a)));
    L.trig_lo[i] = make_float2(static_cast<float>(cosl(b)), static_cast<float>(sinl(b)));
  }
  L.trig_hi[0] = make_float2(1.0f, 0.0f);
  L.trig_hi[1024] = make_float2(0.0f, 1.0f);
  L.trig_hi[2048] = make_float2(-1.0f, 0.0f);
  L.trig_hi[3072] = make_float2(0.0f, -1.0f);
}
// NormalLut2 (see dist_transforms.cuh), long double arithmetic.
static void build_normal_lut2(NormalLut2& L) {
  const long double C2 = static_cast<long double>(kTwoLn2);
  for (int j = 0; j < 2048; ++j) {
    const long double mc = 1.0L + (j + 0.5L) / 2048.0L;     // bucket centre of m
    long double inv = nearbyintl(4096.0L / mc) / 4096.0L;    // multiple of 2^-12
    if (j == 0) inv = 1.0L;                                  // n = 2^24 (k = 0): s = 0, A = 0
    const long double T = (j < 1024) ? 2.0L * logl(inv) : 2.0L * logl(2.0L * inv) - C2;
    L.logt[j].inv = static_cast<float>(inv);
    L.logt[j].pad = 0.0f;
    L.logt[j].T = static_cast<double>(T);
  }
  L.logt[0].T = 0x1p-1000;  // X > 0 at k = 0
#if SDR_N2_COS2
  const long double pi = 3.141592653589793238462643383279502884L;
  for (int i = 0; i < 4096; ++i) {
    const long double a = 2.0L * pi * i / 4096.0L, b = 2.0L * pi * i / 16777216.0L;
    L.cos_hi[i] = make_double2(static_cast<double>(cosl(a)), static_cast<double>(sinl(a)));
    L.cos_lo[i] = make_double2(static_cast<double>(cosl(b)), static_cast<double>(sinl(b)));
  }
  L.cos_hi[0] = make_double2(1.0, 0.0);
  L.cos_hi[1024] = make_double2(0.0, 1.0);
  L.cos_hi[2048] = make_double2(-1.0, 0.0);
  L.cos_hi[3072] = make_double2(0.0, -1.0);
#else
  NormalLut h;
  build_normal_lut(h);
  memcpy(L.trig, h.trig, sizeof(L.trig));
#endif
}
static NormalState g_nm[64];

static int fill_dist_params(const sdr_dist& dist, int dt, DistP& P, int device) {
  memset(static_cast<void*>(&P), 0, sizeof(P));
  P.kind = dist.kind;
  P.ispan = FastDiv64(1);
  switch (dist.kind) {
    case SDR_UNIFORM01:
      if (dt != SDR_F32 && dt != SDR_F64) return SDR_E_DTYPE;
      break;
    case SDR_UNIFORM: {
      const double lo = dist.fparam[0], hi = dist.fparam[1];
      if (!(lo < hi)) return SDR_E_PARAM;
      if (dt != SDR_F32 && dt != SDR_F64 && dt != SDR_BF16 && dt != SDR_F16) return SDR_E_DTYPE;
      // hi - lo is formed in Python float64 then weakly cast (rng.py:138).
      P.lo = lo;
      P.span = hi - lo;
      P.lo32 = static_cast<float>(lo);
      P.span32 = static_cast<float>(hi - lo);
      break;
    }
    case SDR_NORMAL: {
      if (!(dist.fparam[1] > 0)) return SDR_E_PARAM;
      if (dt != SDR_F32 && dt != SDR_F64 && dt != SDR_BF16 && dt != SDR_F16) return SDR_E_DTYPE;
      P.mean = dist.fparam[0];
      P.stdv = dist.fparam[1];
      std::lock_guard<std::mutex> lk(g_nm_mu);
      if (device < 0 || device >= 64 || !g_nm[device].loaded) return SDR_E_NOTABLES;
      P.nm.rtab = g_nm[device].rtab;
      P.nm.ctab = g_nm[device].ctab;
      {
        const NormalState& S = g_nm[device];
        P.nm.em.code_l = S.code;
        P.nm.em.code_c = S.code ? S.code + (1u << 20) : nullptr;
        P.nm.em.xk_l = S.xk;
        P.nm.em.xv_l = S.xv;
        P.nm.em.xk_c = S.xk ? S.xk + S.nx_l : nullptr;
        P.nm.em.xv_c = S.xv ? S.xv + S.nx_l : nullptr;
        P.nm.em.nx_l = S.nx_l;
        P.nm.em.nx_c = S.nx_c;
      }
      P.nm.lut = g_nm[device].lut;
      P.nm.lut32 = g_nm[device].lut32;
      P.nm.lut2 = g_nm[device].lut2;
      {
        const NormalState& S = g_nm[device];
        P.nm.dr = nullptr;
        P.nm.dc = nullptr;
        P.nm.cdd = nullptr;
        if (S.delta != nullptr && S.cmode == 1) {  // dr[2^24], then the 8-bit c_cr corrections (dc8)
          P.nm.dr = reinterpret_cast<const DeltaR*>(S.delta);
          P.nm.cdd = S.cdd;
        } else if (S.delta != nullptr) {           // dc[2^24] (int16), then dr[2^24]
          P.nm.dc = reinterpret_cast<const int16_t*>(S.delta);
          P.nm.dr = reinterpret_cast<const DeltaR*>(S.delta + (sizeof(int16_t) << 24));
        }
      }
      {
        // float64 fast path (see normal_certified): with Er, Ec the calibrated
        // errors of r_fast / c_fast and u = 2^-53,
        //   |v - v_np| <= 2.03u|v| + (std r)(Er' + Ec(1 + Er') + 2.01u)/(1 - Er'),
        // Er' = Er/(1-Er) + 8u (std folded into the Newton step); doubled.
        // k = 0 (r_np = 0, r_fast <= 2^-490) is covered by k0.
        const double u = 0x1p-53, Er = g_nm[device].err_r, Ec = g_nm[device].err_c;
        const double Erp = (Er / (1.0 - Er) + 8.0 * u) * (1.0 + 0x1p-30);
        P.nm.nh = -0.5 * P.stdv;
        P.nm.th = 1.5 * P.stdv;
        P.nm.kr = 2.0 * (Erp + Ec * (1.0 + Erp) + 2.01 * u) / (1.0 - Erp) * (1.0 + 0x1p-30);
        P.nm.k0 = 2.0 * fabs(P.stdv) * 0x1p-489 + 0x1p-1060;
        // the kernel's B = rs kr + k0 also covers |v| 2^-51 <= (|mean| + rs (1 + 2^-48)) 2^-51
        P.nm.kr += 0x1p-51 * (1.0 + 0x1p-40);
        P.nm.k0 += fabs(P.mean) * 0x1p-51 * (1.0 + 0x1p-40);
        if (!(Er < 0x1p-20) || !(Ec < 0x1p-20)) P.nm.kr = INFINITY;  // calibration failed: exact path
        {  // the same bound for the NormalLut2 functions (r_fast2 / c_fast2)
          const double Er2 = g_nm[device].err_r2, Ec2 = g_nm[device].err_c2;
          const double Erp2 = (Er2 / (1.0 - Er2) + 8.0 * u) * (1.0 + 0x1p-30);
          P.nm.kr2 = 2.0 * (Erp2 + Ec2 * (1.0 + Erp2) + 2.01 * u) / (1.0 - Erp2) * (1.0 + 0x1p-30) +
                     0x1p-51 * (1.0 + 0x1p-40);
          P.nm.k02 = P.nm.k0;
          if (!(Er2 < 0x1p-20) || !(Ec2 < 0x1p-20)) P.nm.kr2 = INFINITY;
        }
        // float32 path (bfloat16 outputs): Er32, Ec32 the calibrated errors of
        // r32_fast / c32_fast;  |v32 - v_np| <= |std| r (Er32 + Ec32(1+Er32) + 2^-23)
        // + 2^-24 (|v32| + |mean|) + |std| 2^-49 (k = 0), doubled.
        const double Er32 = g_nm[device].err_r32, Ac32 = g_nm[device].err_c32;
        P.nm.err_r32 = Er32;
        P.nm.err_c32 = Ac32;
        P.nm.mean32 = static_cast<float>(P.mean);
        P.nm.std32 = static_cast<float>(P.stdv);
        P.nm.b32_r = static_cast<float>(2.04 * fabs(P.stdv) * (Er32 + Ac32 * (1.0 + Er32) + 0x1p-23) + 0x1p-60);
        P.nm.b32_c = static_cast<float>(2.04 * 0x1p-24 * fabs(P.mean) + 2.0 * fabs(P.stdv) * 0x1p-48 + 0x1p-140);
        // B32 = r b32_r + b32_c also covers |v| 2^-22 <= (|mean32| + std32 r (1 + 2^-21)) 2^-22
        P.nm.b32_r = static_cast<float>(P.nm.b32_r + fabs(static_cast<double>(P.nm.std32)) * 0x1p-22 * (1.0 + 0x1p-20));
        P.nm.b32_c = static_cast<float>(P.nm.b32_c + fabs(static_cast<double>(P.nm.mean32)) * 0x1p-22 * (1.0 + 0x1p-20));
        if (!(Er32 < 0x1p-12) || !(Ac32 < 0x1p-12)) P.nm.b32_r = INFINITY;  // calibration failed
        {  // r32_mufu: |r - r_np| <= Erm r + Eim h (h = 1/r to 2^-21); c32_fast: |c - c_np| <= Ac32;
           // |v32 - v_np| <= |std| (r (Erm + Ac32 (1 + Erm) + 2^-23) + Eim h (1 + 2^-20)(1 + Ac32))
           //                + the b32_c / |v| 2^-22 terms of the table path, doubled (x2.04).
          const double Erm = g_nm[device].err_rm, Eim = g_nm[device].err_im;
          P.nm.bm_r = static_cast<float>(2.04 * fabs(P.stdv) * (Erm + Ac32 * (1.0 + Erm) + 0x1p-23) + 0x1p-60 +
                                         fabs(static_cast<double>(P.nm.std32)) * 0x1p-22 * (1.0 + 0x1p-20));
          P.nm.bm_i = static_cast<float>(2.04 * fabs(P.stdv) * Eim * (1.0 + 0x1p-20) * (1.0 + Ac32) + 0x1p-140);
          P.nm.bm_c = P.nm.b32_c;
          const double Acm = g_nm[device].err_cm;  // the same bound with the MUFU cosine
          P.nm.bmc_r = static_cast<float>(2.04 * fabs(P.stdv) * (Erm + Acm * (1.0 + Erm) + 0x1p-23) + 0x1p-60 +
                                          fabs(static_cast<double>(P.nm.std32)) * 0x1p-22 * (1.0 + 0x1p-20));
          P.nm.bmc_i = static_cast<float>(2.04 * fabs(P.stdv) * Eim * (1.0 + 0x1p-20) * (1.0 + Acm) + 0x1p-140);
          if (!(Acm < 0x1p-12)) P.nm.bmc_r = INFINITY;
          if (!(Erm < 0x1p-12) || !(Eim < 0x1p-12) || !(P.nm.b32_r < INFINITY))
            P.nm.bm_r = P.nm.bmc_r = INFINITY;  // calibration failed: every element takes the float64 path
        }
        // Test hook: SDR_NORMAL_PATH=exact sends every element through the NumPy
        // tables, =f64 skips the float32 path (results must be identical).
        if (const char* path = getenv("SDR_NORMAL_PATH")) {
          if (strcmp(path, "exact") == 0) {
            P.nm.kr = P.nm.kr2 = P.nm.b32_r = P.nm.bm_r = P.nm.bmc_r = INFINITY;
            P.nm.dr = nullptr;
            P.nm.dc = nullptr;
          }
          if (strcmp(path, "f64") == 0) P.nm.b32_r = P.nm.bm_r = P.nm.bmc_r = INFINITY;
        }
      }
      P.nm.fallbacks = g_nm[device].fallbacks;
      break;
    }
    case SDR_RANDINT: {
      const int64_t lo = dist.iparam[0], hi = dist.iparam[1];
      if (!(lo < hi)) return SDR_E_PARAM;
      if (dt != SDR_I64 && dt != SDR_I32 && dt != SDR_F64 && dt != SDR_F32) return SDR_E_DTYPE;
      P.ilo = lo;
      P.ispan = FastDiv64(static_cast<uint64_t>(hi) - static_cast<uint64_t>(lo));
      break;
    }
    case SDR_BERNOULLI: {
      const double p = dist.fparam[0];
      if (!(p >= 0.0 && p <= 1.0)) return SDR_E_PARAM;
      // u < p  <=>  k53 < ceil(p * 2^53)  <=>  u64 < ceil(p*2^53) << 11.
      const double t = ceil(p * 9007199254740992.0);
      const uint64_t T = static_cast<uint64_t>(t);
      P.keep_all = (T >= (uint64_t{1} << 53)) ? 1u : 0u;
      P.keep_thr = P.keep_all ? 0 : (T << 11);
      break;
    }
    default:
      return SDR_E_DIST;
  }
  return SDR_OK;
}

// Dynamic shared memory of the fill kernels (the float32 Normal tables exceed
// the 48 KiB static limit), with the opt-in attribute set before each launch.
template <int DIST, int DT>
static constexpr size_t fill_dyn_smem() {
  return uses_lut2<DIST, DT>() ? sizeof(NormalLut2)
         : (DIST == SDR_NORMAL && half_dt<DT>() && SDR_NORMAL_BF16_F32 && !tablefree<DIST, DT>())
               ? sizeof(NormalLut32) : 0;
}
template <typename K>
static void allow_dyn_smem(K kernel, size_t bytes) {
  if (bytes > 48 * 1024) cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes));
}
// float64 Normal kernels read c_cr's 64 KiB table through L1: ask for the
// smallest shared-memory carve-out that holds their two CTAs' static tables.
#ifndef SDR_F64_CARVEOUT
#define SDR_F64_CARVEOUT 40
#endif
template <int DIST, int DT, typename K>
static void prefer_l1(K kernel) {
  if constexpr (DIST == SDR_NORMAL && DT == SDR_F64 && SDR_F64_CARVEOUT > 0) {
    static std::atomic<uint64_t> done{0};  // once per (kernel, device)
    int dev = 0;
    cudaGetDevice(&dev);
    const uint64_t bit = uint64_t{1} << (dev & 63);
    if ((done.load(std::memory_order_relaxed) & bit) == 0) {
      cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout, SDR_F64_CARVEOUT);
      done.fetch_or(bit, std::memory_order_relaxed);
    }
  }
}

template <int DIST, int DT>
static void launch_fill(const FillArgs& A0, bool fast, cudaStream_t s) {
  FillArgs A = A0;
  constexpr size_t dsm = fill_dyn_smem<DIST, DT>();
  constexpr int nt = fill_threads<DIST, DT>();
  if (fast && A.aligned) {
    allow_dyn_smem(k_fill_fast<DIST, DT, true>, dsm);
    prefer_l1<DIST, DT>(k_fill_fast<DIST, DT, true>);
    const int grid = grid_for(k_fill_fast<DIST, DT, true>, A.nchunks, nt, dsm);
    set_walk(A.walk, A.ix.cv, A.chunks_per_row, static_cast<uint64_t>(grid) * nt, kV);
    launch_pdl(k_fill_fast<DIST, DT, true>, grid, s, A, dsm, nt);
  } else if (fast) {
    allow_dyn_smem(k_fill_fast<DIST, DT, false>, dsm);
    prefer_l1<DIST, DT>(k_fill_fast<DIST, DT, false>);
    const int grid = grid_for(k_fill_fast<DIST, DT, false>, A.nchunks, nt, dsm);
    set_walk(A.walk, A.ix.cv, A.chunks_per_row, static_cast<uint64_t>(grid) * nt, kV);
    launch_pdl(k_fill_fast<DIST, DT, false>, grid, s, A, dsm, nt);
  } else {
    k_fill_generic<DIST, DT><<<grid_for(k_fill_generic<DIST, DT>, A.ix.cv.numel, 256), 256, 0, s>>>(A);
  }
}

template <int DIST>
static int dispatch_fill_dt(int dt, const FillArgs& A, bool fast, cudaStream_t s) {
  switch (dt) {
    case SDR_F32: launch_fill<DIST, SDR_F32>(A, fast, s); break;
    case SDR_F64: launch_fill<DIST, SDR_F64>(A, fast, s); break;
    case SDR_BF16:
      if constexpr (DIST != SDR_UNIFORM01 && DIST != SDR_RANDINT) launch_fill<DIST, SDR_BF16>(A, fast, s);
      else return SDR_E_DTYPE;
      break;
    case SDR_F16:
      if constexpr (DIST != SDR_UNIFORM01 && DIST != SDR_RANDINT) launch_fill<DIST, SDR_F16>(A, fast, s);
      else return SDR_E_DTYPE;
      break;
    case SDR_I64:
      if constexpr (DIST == SDR_RANDINT || DIST == SDR_BERNOULLI) launch_fill<DIST, SDR_I64>(A, fast, s);
      else return SDR_E_DTYPE;
      break;
    case SDR_I32:
      if constexpr (DIST == SDR_RANDINT || DIST == SDR_BERNOULLI) launch_fill<DIST, SDR_I32>(A, fast, s);
      else return SDR_E_DTYPE;
      break;
    case SDR_U8:
      if constexpr (DIST == SDR_BERNOULLI) launch_fill<DIST, SDR_U8>(A, fast, s);
      else return SDR_E_DTYPE;
      break;
    case SDR_BOOL:
      if constexpr (DIST == SDR_BERNOULLI) launch_fill<DIST, SDR_BOOL>(A, fast, s);
      else return SDR_E_DTYPE;
      break;
    default:
      return SDR_E_DTYPE;
  }
  return check_launch();
}


int fill(void* out, int dt, const sdr_dist& dist, const sdr_rng& rng, const sdr_view& view,
         cudaStream_t s) {
  if (rng.theta < 1) return SDR_E_INVALID;
  if (dtype_size(dt) == 0) return SDR_E_DTYPE;
  CanonView cv;
  int st = canonicalize(view, cv);
  if (st != SDR_OK) return st;
  int dev = 0;
  cudaGetDevice(&dev);
  FillArgs A;
  memset(static_cast<void*>(&A), 0, sizeof(A));
  st = fill_dist_params(dist, dt, A.d, dev);
  if (st != SDR_OK) return st;
  if (cv.numel == 0) return SDR_OK;
  if (out == nullptr) return SDR_E_INVALID;
  A.g = make_gen(rng);
  A.ix = make_indexer(cv);
  A.out = out;
  bool fast = cv.istride == 1 && cv.inner % kV == 0 && aligned16(out);
  setup_chunks(cv, fast, A.nchunks, A.chunks_per_row, A.div_cpr);
  A.aligned = fast && chunks_aligned(cv, rng.theta, kV);
  if (!fast && cv.istride == 1 && cv.inner >= kV) {  // ragged rows: chunked, per-element stores
    fast = true;
    A.ragged = 1;
    A.chunks_per_row = (static_cast<uint64_t>(cv.inner) + kV - 1) / kV;
    A.nchunks = static_cast<uint64_t>(cv.numel / cv.inner) * A.chunks_per_row;
    A.div_cpr = FastDiv64(A.chunks_per_row);
    A.aligned = chunks_aligned(cv, rng.theta, kV);
  }
  switch (dist.kind) {
    case SDR_UNIFORM01: return dispatch_fill_dt<SDR_UNIFORM01>(dt, A, fast, s);
    case SDR_UNIFORM: return dispatch_fill_dt<SDR_UNIFORM>(dt, A, fast, s);
    case SDR_NORMAL: return dispatch_fill_dt<SDR_NORMAL>(dt, A, fast, s);
    case SDR_RANDINT: return dispatch_fill_dt<SDR_RANDINT>(dt, A, fast, s);
    case SDR_BERNOULLI: return dispatch_fill_dt<SDR_BERNOULLI>(dt, A, fast, s);
    default: return SDR_E_DIST;
  }
}

// Calls f(std::integral_constant<int, DT>) for the output dtypes the
// reference's NumPy/ml_dtypes path gives distribution DIST; SDR_E_DTYPE else.
template <int DIST, typename F>
static int with_dtype(int dt, F&& f) {
  constexpr bool flt = true, half = DIST != SDR_UNIFORM01 && DIST != SDR_RANDINT;
  constexpr bool ints = DIST == SDR_RANDINT || DIST == SDR_BERNOULLI, bytes = DIST == SDR_BERNOULLI;
  switch (dt) {
    case SDR_F32: if constexpr (flt) return f(std::integral_constant<int, SDR_F32>{}); break;
    case SDR_F64: if constexpr (flt) return f(std::integral_constant<int, SDR_F64>{}); break;
    case SDR_BF16: if constexpr (half) return f(std::integral_constant<int, SDR_BF16>{}); break;
    case SDR_F16: if constexpr (half) return f(std::integral_constant<int, SDR_F16>{}); break;
    case SDR_I64: if constexpr (ints) return f(std::integral_constant<int, SDR_I64>{}); break;
    case SDR_I32: if constexpr (ints) return f(std::integral_constant<int, SDR_I32>{}); break;
    case SDR_U8: if constexpr (bytes) return f(std::integral_constant<int, SDR_U8>{}); break;
    case SDR_BOOL: if constexpr (bytes) return f(std::integral_constant<int, SDR_BOOL>{}); break;
    default: break;
  }
  return SDR_E_DTYPE;
}

template <typename F>
static int with_dist(int kind, F&& f) {
  switch (kind) {
    case SDR_UNIFORM01: return f(std::integral_constant<int, SDR_UNIFORM01>{});
    case SDR_UNIFORM: return f(std::integral_constant<int, SDR_UNIFORM>{});
    case SDR_NORMAL: return f(std::integral_constant<int, SDR_NORMAL>{});
    case SDR_RANDINT: return f(std::integral_constant<int, SDR_RANDINT>{});
    case SDR_BERNOULLI: return f(std::integral_constant<int, SDR_BERNOULLI>{});
    default: return SDR_E_DIST;
  }
}

int transform(const uint32_t* w0, const uint32_t* w1, int64_t n, const sdr_dist& dist, void* out,
              int dt, cudaStream_t s) {
  if (n < 0) return SDR_E_INVALID;
  if (dtype_size(dt) == 0) return SDR_E_DTYPE;
  int dev = 0;
  cudaGetDevice(&dev);
  DistP P;
  const int st = fill_dist_params(dist, dt, P, dev);
  if (st != SDR_OK) return st;
  if (n == 0) return SDR_OK;
  if (w0 == nullptr || w1 == nullptr || out == nullptr) return SDR_E_INVALID;
  return with_dist(dist.kind, [&](auto dk) {
    constexpr int DIST = decltype(dk)::value;
    return with_dtype<DIST>(dt, [&](auto dtc) {
      constexpr int DT = decltype(dtc)::value;
      const int grid = grid_for(k_transform<DIST, DT>, static_cast<uint64_t>(n), 256);
      k_transform<DIST, DT><<<grid, 256, 0, s>>>(w0, w1, n, P, out);
      return check_launch();
    });
  });
}

int philox_blocks(const uint64_t* tau, const uint64_t* beta, int64_t n, uint64_t seed,
                  uint32_t* words, cudaStream_t s) {
  if (n < 0) return SDR_E_INVALID;
  if (n == 0) return SDR_OK;
  const RoundKeys K = make_keys(seed);
  k_philox_blocks<<<static_cast<unsigned>((n + 255) / 256), 256, 0, s>>>(tau, beta, n, K, words);
  return check_launch();
}

// Build the per-device Normal mirror from the host NumPy tables L[k] =
// log1p(-k 2^-24) and C[k] = cos((2 pi)(k 2^-24)): the full tables are
// uploaded only transiently, to (1) derive the 2-bit corrections against the
// device libm (ExactMirror), (2) verify that mirror on all 2^24 points of both
// functions, and (3) calibrate the fast paths exhaustively.  Resident after
// load: the 8 MiB of codes + exceptions (or, if verification failed, the full
// tables as before) and the small fast-path LUTs.
int normal_tables_load(int device, const double* l_host, const double* c_host, double* er,
                       double* ec) {
  if (device < 0 || device >= 64 || l_host == nullptr || c_host == nullptr) return SDR_E_INVALID;
  std::lock_guard<std::mutex> lk(g_nm_mu);
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(device);
  NormalState& S = g_nm[device];
  const size_t bytes = sizeof(double) << 24;
  const unsigned int cap = 1u << 20;  // exception capacity per function
  cudaEvent_t t0, t1;
  cudaEventCreate(&t0);
  cudaEventCreate(&t1);
  cudaEventRecord(t0);
  cudaError_t e = cudaSuccess;
  if (S.lut == nullptr) {
    e = cudaMalloc(&S.fallbacks, 10 * sizeof(unsigned long long));
    if (e == cudaSuccess) e = cudaMalloc(&S.lut, sizeof(NormalLut));
    if (e == cudaSuccess) e = cudaMalloc(&S.lut32, sizeof(NormalLut32));
    if (e == cudaSuccess) e = cudaMalloc(&S.lut2, sizeof(NormalLut2));
    if (e == cudaSuccess) {
      NormalLut h;
      build_normal_lut(h);
      NormalLut32 h32;
      build_normal_lut32(h, h32);
      std::vector<NormalLut2> h2(1);
      build_normal_lut2(h2[0]);
      e = cudaMemcpy(S.lut, &h, sizeof(NormalLut), cudaMemcpyHostToDevice);
      if (e == cudaSuccess) e = cudaMemcpy(S.lut32, &h32, sizeof(NormalLut32), cudaMemcpyHostToDevice);
      if (e == cudaSuccess) e = cudaMemcpy(S.lut2, h2.data(), sizeof(NormalLut2), cudaMemcpyHostToDevice);
    }
  }
  // a reload replaces the previous mirror
  cudaFree(S.delta);
  S.delta = nullptr;
  cudaFree(S.cdd);
  S.cdd = nullptr;
  S.cmode = 0;
  cudaFree(S.rtab);
  cudaFree(S.ctab);
  cudaFree(S.code);
  cudaFree(S.xk);
  cudaFree(S.xv);
  S.rtab = S.ctab = nullptr;
  S.code = S.xk = nullptr;
  S.xv = nullptr;
  S.nx_l = S.nx_c = 0;
  S.loaded = false;
  double *dl = nullptr, *dc = nullptr, *xv = nullptr;
  uint32_t* xk = nullptr;
  unsigned int* counts = nullptr;
  if (e == cudaSuccess) e = cudaMalloc(&dl, bytes);
  if (e == cudaSuccess) e = cudaMalloc(&dc, bytes);
  if (e == cudaSuccess) e = cudaMemcpy(dl, l_host, bytes, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(dc, c_host, bytes, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemset(S.fallbacks, 0, 10 * sizeof(unsigned long long));
  // (3) calibration of the fast paths against the full tables
  if (e == cudaSuccess) {
    k_normal_calibrate<<<(1u << 24) / 256, 256>>>(dl, dc, S.lut, S.lut32, S.lut2, S.fallbacks + 1,
                                                  S.fallbacks + 2);
    k_normal_calibrate_mufu<<<(1u << 24) / 256, 256>>>(dl, dc, S.fallbacks + 7);
    e = cudaGetLastError();
  }
  // (1) codes + unsorted exceptions
  if (e == cudaSuccess) e = cudaMalloc(&S.code, 2 * sizeof(uint32_t) << 20);
  if (e == cudaSuccess) e = cudaMalloc(&xk, 2 * sizeof(uint32_t) * cap);
  if (e == cudaSuccess) e = cudaMalloc(&xv, 2 * sizeof(double) * cap);
  if (e == cudaSuccess) e = cudaMalloc(&counts, 2 * sizeof(unsigned int));
  if (e == cudaSuccess) e = cudaMemset(counts, 0, 2 * sizeof(unsigned int));
  if (e == cudaSuccess) {
    k_mirror_codes<<<(1u << 20) / 256, 256>>>(dl, dc, S.code, S.code + (1u << 20), xk, xv, xk + cap,
                                              xv + cap, counts, cap);
    e = cudaGetLastError();
  }
  unsigned int nx[2] = {0, 0};
  if (e == cudaSuccess) e = cudaMemcpy(nx, counts, sizeof(nx), cudaMemcpyDeviceToHost);
  bool compact = e == cudaSuccess && nx[0] <= cap && nx[1] <= cap;
  if (compact && nx[0] + nx[1] > 0) {  // sort each list by key on the host, upload packed
    std::vector<uint32_t> hk(2 * cap);
    std::vector<double> hv(2 * cap);
    e = cudaMemcpy(hk.data(), xk, 2 * sizeof(uint32_t) * cap, cudaMemcpyDeviceToHost);
    if (e == cudaSuccess) e = cudaMemcpy(hv.data(), xv, 2 * sizeof(double) * cap, cudaMemcpyDeviceToHost);
    std::vector<uint32_t> sk;
    std::vector<double> sv;
    for (int f = 0; f < 2 && e == cudaSuccess; ++f) {
      std::vector<std::pair<uint32_t, double>> kv(nx[f]);
      for (unsigned int i = 0; i < nx[f]; ++i) kv[i] = {hk[f * cap + i], hv[f * cap + i]};
      std::sort(kv.begin(), kv.end(), [](const auto& a, const auto& b) { return a.first < b.first; });
      for (const auto& p : kv) {
        sk.push_back(p.first);
        sv.push_back(p.second);
      }
    }
    if (e == cudaSuccess) e = cudaMalloc(&S.xk, sk.size() * sizeof(uint32_t));
    if (e == cudaSuccess) e = cudaMalloc(&S.xv, sv.size() * sizeof(double));
    if (e == cudaSuccess) e = cudaMemcpy(S.xk, sk.data(), sk.size() * sizeof(uint32_t), cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(S.xv, sv.data(), sv.size() * sizeof(double), cudaMemcpyHostToDevice);
  }
  S.nx_l = static_cast<int>(nx[0]);
  S.nx_c = static_cast<int>(nx[1]);
  // (2) exhaustive verification of the compact mirror
  unsigned long long bad = ~0ull;
  if (compact && e == cudaSuccess) {
    ExactMirror M{S.code, S.code + (1u << 20), S.xk, S.xv, S.xk ? S.xk + S.nx_l : nullptr,
                  S.xv ? S.xv + S.nx_l : nullptr, S.nx_l, S.nx_c};
    e = cudaMemset(S.fallbacks, 0, sizeof(unsigned long long));
    if (e == cudaSuccess) {
      k_mirror_verify<<<(1u << 24) / 256, 256>>>(M, dl, dc, S.fallbacks);
      e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaMemcpy(&bad, S.fallbacks, sizeof(bad), cudaMemcpyDeviceToHost);
    if (e == cudaSuccess) e = cudaMemset(S.fallbacks, 0, sizeof(unsigned long long));
  }
  compact = compact && bad == 0;
  if (e == cudaSuccess && !compact) {  // keep the full tables (r derived from L on the device)
    k_r_from_l<<<(1u << 24) / 256, 256>>>(dl);
    e = cudaGetLastError();
    S.rtab = dl;
    S.ctab = dc;
    dl = dc = nullptr;
    cudaFree(S.code);
    cudaFree(S.xk);
    cudaFree(S.xv);
    S.code = S.xk = nullptr;
    S.xv = nullptr;
  }
  // float64 corrections against whichever exact form is resident
  // (SDR_NORMAL_F64_DELTA=0: float64 outputs take the mirror per element)
  const char* dflag = getenv("SDR_NORMAL_F64_DELTA");
  if (e == cudaSuccess && !(dflag != nullptr && strcmp(dflag, "0") == 0)) {
    unsigned long long* st = nullptr;
    ExactMirror M{S.code, S.code ? S.code + (1u << 20) : nullptr, S.xk, S.xv,
                  S.xk ? S.xk + S.nx_l : nullptr, S.xv ? S.xv + S.nx_l : nullptr, S.nx_l, S.nx_c};
    e = cudaMalloc(&st, 8 * sizeof(unsigned long long));
    if (e == cudaSuccess) e = cudaMemset(st, 0, 8 * sizeof(unsigned long long));
    // cosine: c_cr where it verifies on every point (cmode 1), else 16-bit corrections of c_fast
    const char* cflag = getenv("SDR_NORMAL_COS_CR");
    bool cr = e == cudaSuccess && !(cflag != nullptr && strcmp(cflag, "0") == 0);
    if (cr) {
      std::vector<CosDD> h(kCosDD);
      build_cos_dd(h.data());
      e = cudaMalloc(&S.delta, kDeltaBytesCr);
      if (e == cudaSuccess) e = cudaMalloc(&S.cdd, kCosDD * sizeof(CosDD));
      if (e == cudaSuccess) e = cudaMemcpy(S.cdd, h.data(), kCosDD * sizeof(CosDD), cudaMemcpyHostToDevice);
      if (e == cudaSuccess) {
        NormalMirror NM;
        memset(static_cast<void*>(&NM), 0, sizeof(NM));
        NM.cdd = S.cdd;
        k_normal_cos_cr<<<(1u << 24) / 256, 256>>>(M, S.ctab, NM, reinterpret_cast<int8_t*>(S.delta + (sizeof(DeltaR) << 24)),
                                                    st + 4);
        k_normal_deltas<<<(1u << 24) / 256, 256>>>(M, S.rtab, S.ctab, S.lut, reinterpret_cast<DeltaR*>(S.delta),
                                                    nullptr, st);
        e = cudaGetLastError();
      }
      if (e == cudaSuccess) e = cudaMemcpy(S.cr_stats, st + 4, sizeof(S.cr_stats), cudaMemcpyDeviceToHost);
      cr = e == cudaSuccess && S.cr_stats[2] == 0;
      if (cr) {
        S.cmode = 1;
      } else {
        cudaFree(S.delta);
        cudaFree(S.cdd);
        S.delta = nullptr;
        S.cdd = nullptr;
        if (e == cudaSuccess) e = cudaMemset(st, 0, 8 * sizeof(unsigned long long));
      }
    }
    if (!cr && e == cudaSuccess) {
      S.cmode = 0;
      e = cudaMalloc(&S.delta, kDeltaBytes);
      if (e == cudaSuccess) {
        k_normal_deltas<<<(1u << 24) / 256, 256>>>(M, S.rtab, S.ctab, S.lut,
                                                    reinterpret_cast<DeltaR*>(S.delta + (sizeof(int16_t) << 24)),
                                                    reinterpret_cast<int16_t*>(S.delta), st);
        e = cudaGetLastError();
      }
    }
    if (e == cudaSuccess) e = cudaMemcpy(S.delta_stats, st, sizeof(S.delta_stats), cudaMemcpyDeviceToHost);
    cudaFree(st);
    if (e != cudaSuccess) {
      cudaFree(S.delta);
      cudaFree(S.cdd);
      S.delta = nullptr;
      S.cdd = nullptr;
      S.cmode = 0;
    }
  }
  // fallbacks[1..6] = max err of r, c (NormalLut), r32, c32 (float32 path), r2, c2 (NormalLut2);
  // [7..9] = Er, Ei of r32_mufu, Ac of c32_mufu
  unsigned long long bits[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
  if (e == cudaSuccess) e = cudaMemcpy(bits, S.fallbacks + 1, 9 * sizeof(bits[0]), cudaMemcpyDeviceToHost);
  cudaFree(dl);
  cudaFree(dc);
  cudaFree(xk);
  cudaFree(xv);
  cudaFree(counts);
  cudaEventRecord(t1);
  cudaEventSynchronize(t1);
  float ms = 0;
  cudaEventElapsedTime(&ms, t0, t1);
  cudaEventDestroy(t0);
  cudaEventDestroy(t1);
  cudaSetDevice(prev);
  if (e != cudaSuccess) {
    set_cuda_error(e);
    return SDR_E_CUDA;
  }
  memcpy(&S.err_r, &bits[0], 8);
  memcpy(&S.err_c, &bits[1], 8);
  memcpy(&S.err_r32, &bits[2], 8);
  memcpy(&S.err_c32, &bits[3], 8);
  memcpy(&S.err_r2, &bits[4], 8);
  memcpy(&S.err_c2, &bits[5], 8);
  memcpy(&S.err_rm, &bits[6], 8);
  memcpy(&S.err_im, &bits[7], 8);
  memcpy(&S.err_cm, &bits[8], 8);
  S.build_ms = ms;
  S.device_bytes = compact ? (2 * sizeof(uint32_t) << 20) + (S.nx_l + S.nx_c) * (sizeof(uint32_t) + sizeof(double))
                           : 2 * bytes;
  S.device_bytes += sizeof(NormalLut) + sizeof(NormalLut32) + sizeof(NormalLut2) + 7 * sizeof(unsigned long long);
  if (getenv("SDR_NORMAL_DEBUG"))
    fprintf(stderr,
            "sdr normal mirror: %s, exceptions log1p %d cos %d, verify-mismatch %llu, %.1f ms, %.2f MiB resident;"
             " calibration r %.3g c %.3g r32 %.3g c32 %.3g r2 %.3g c2 %.3g r32m %.3g / %.3g h c32m %.3g\n",
            compact ? "compact" : "full tables", S.nx_l, S.nx_c, bad, ms, S.device_bytes / 1048576.0, S.err_r,
            S.err_c, S.err_r32, S.err_c32, S.err_r2, S.err_c2, S.err_rm, S.err_im, S.err_cm);
  if (getenv("SDR_NORMAL_DEBUG"))
    fprintf(stderr,
            "sdr normal float64 corrections: %s, cosine %s (tau %.3f: flagged %llu, escapes %llu, unflagged"
            " mismatches %llu, max |d| %llu), escapes r %llu c %llu, max |d| r %llu c %llu\n",
            S.delta ? "built" : "off", S.cmode == 1 ? "c_cr" : "c_fast + 16-bit", SDR_COS_TAU, S.cr_stats[0],
            S.cr_stats[1], S.cr_stats[2], S.cr_stats[3], S.delta_stats[0], S.delta_stats[1], S.delta_stats[2],
            S.delta_stats[3]);
  S.loaded = true;
  if (er) *er = S.err_r;
  if (ec) *ec = S.err_c;
  return SDR_OK;
}

int normal_mirror_info(int device, uint64_t* device_bytes, uint64_t* exceptions, int32_t* compact,
                       double* build_ms) {
  std::lock_guard<std::mutex> lk(g_nm_mu);
  if (device < 0 || device >= 64 || !g_nm[device].loaded) return SDR_E_NOTABLES;
  const NormalState& S = g_nm[device];
  if (device_bytes) *device_bytes = S.device_bytes;
  if (exceptions) *exceptions = static_cast<uint64_t>(S.nx_l + S.nx_c);
  if (compact) *compact = S.rtab == nullptr ? 1 : 0;
  if (build_ms) *build_ms = S.build_ms;
  return SDR_OK;
}

int normal_delta_info(int device, uint64_t* device_bytes, uint64_t* escapes_r, uint64_t* escapes_c,
                      uint64_t* max_abs_r, uint64_t* max_abs_c) {
  std::lock_guard<std::mutex> lk(g_nm_mu);
  if (device < 0 || device >= 64 || !g_nm[device].loaded) return SDR_E_NOTABLES;
  const NormalState& S = g_nm[device];
  const bool on = S.delta != nullptr;
  const bool cr = on && S.cmode == 1;
  if (device_bytes) *device_bytes = on ? (cr ? kDeltaBytesCr + kCosDD * sizeof(CosDD) : kDeltaBytes) : 0;
  if (escapes_r) *escapes_r = on ? S.delta_stats[0] : 0;
  if (escapes_c) *escapes_c = on ? (cr ? S.cr_stats[1] : S.delta_stats[1]) : 0;
  if (max_abs_r) *max_abs_r = on ? S.delta_stats[2] : 0;
  if (max_abs_c) *max_abs_c = on ? (cr ? S.cr_stats[3] : S.delta_stats[3]) : 0;
  return SDR_OK;
}

int normal_tables_loaded(int device) {
  std::lock_guard<std::mutex> lk(g_nm_mu);
  return (device >= 0 && device < 64 && g_nm[device].loaded) ? 1 : 0;
}

int normal_fallback_count(int device, uint64_t* count) {
  std::lock_guard<std::mutex> lk(g_nm_mu);
  if (device < 0 || device >= 64 || !g_nm[device].loaded || count == nullptr) return SDR_E_NOTABLES;
  unsigned long long c = 0;
  cudaError_t e = cudaMemcpy(&c, g_nm[device].fallbacks, sizeof(c), cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) {
    set_cuda_error(e);
    return SDR_E_CUDA;
  }
  *count = c;
  return SDR_OK;
}

// Descriptor upload: the batch's FillArgs travel as kernel parameters (up to
// kUploadN per launch, 29 KB) and are copied into the stream-ordered device
// table by a tiny kernel, so the whole batched fill -- allocation, upload,
// fill, free -- is stream-ordered and can be captured in a CUDA graph (no
// pageable host copy).
constexpr int kUploadN = 24;
struct UploadArgs {
  FillArgs a[kUploadN];
  uint64_t prefix[kUploadN];
  FillArgs* dst;
  uint64_t* dst_prefix;
  uint64_t* counter;  // the batch kernel's tile counter (zeroed by the first upload), or null
  int n;
};
static_assert(sizeof(UploadArgs) <= 32000, "kernel parameter limit");

__global__ void __launch_bounds__(256) k_upload_descs(const __grid_constant__ UploadArgs U) {
  const int words = U.n * static_cast<int>(sizeof(FillArgs) / 16);
  const uint4* src = reinterpret_cast<const uint4*>(U.a);
  uint4* dst = reinterpret_cast<uint4*>(U.dst);
  for (int w = threadIdx.x; w < words; w += blockDim.x) dst[w] = src[w];
  if (threadIdx.x < U.n) U.dst_prefix[threadIdx.x] = U.prefix[threadIdx.x];
  if (threadIdx.x == 0 && U.counter != nullptr) *U.counter = 0;
}

template <int DIST, int DT>
static void launch_batch(const FillArgs* d_descs, const uint64_t* d_prefix, int n, uint64_t ntiles,
                         cudaStream_t s) {
  constexpr size_t dsm = fill_dyn_smem<DIST, DT>();
  constexpr int nt = fill_threads<DIST, DT>();
  allow_dyn_smem(k_fill_batch<DIST, DT>, dsm);
  prefer_l1<DIST, DT>(k_fill_batch<DIST, DT>);
  // persistent: one wave of resident CTAs (SMs x occupancy) taking tiles from
  // the counter at d_prefix[n]
  const int grid = grid_for(k_fill_batch<DIST, DT>, ntiles * nt, nt, dsm);
  k_fill_batch<DIST, DT><<<grid, nt, dsm, s>>>(d_descs, d_prefix, n, ntiles,
                                               reinterpret_cast<unsigned long long*>(const_cast<uint64_t*>(d_prefix + n)));
}

// SDR_OK when distribution `kind` can produce dtype `dt` (the reference's
// NumPy / ml_dtypes casts), else SDR_E_DTYPE / SDR_E_DIST.
static int dist_dtype_ok(int kind, int dt) {
  return with_dist(kind, [&](auto D) { return with_dtype<decltype(D)::value>(dt, [](auto) { return SDR_OK; }); });
}

int fill_batch(void* const* outs, const int32_t* dts, const sdr_dist* dists, const sdr_rng* rngs,
               const sdr_view* views, int n, cudaStream_t s) {
  if (n < 0 || (n > 0 && (outs == nullptr || dts == nullptr || dists == nullptr ||
                          rngs == nullptr || views == nullptr)))
    return SDR_E_INVALID;
  int dev = 0;
  cudaGetDevice(&dev);
  // Validate everything first; group members by (distribution kind, dtype).
  struct Member { FillArgs a; uint64_t tiles; };
  std::vector<std::vector<Member>> groups(5 * 8);
  for (int i = 0; i < n; ++i) {
    if (rngs[i].theta < 1) return SDR_E_INVALID;
    const int dt = dts[i];
    if (dtype_size(dt) == 0 || dists[i].kind < 0 || dists[i].kind > 4) return SDR_E_DTYPE;
    int st = dist_dtype_ok(dists[i].kind, dt);
    if (st != SDR_OK) return st;
    CanonView cv;
    st = canonicalize(views[i], cv);
    if (st != SDR_OK) return st;
    Member m;
    memset(static_cast<void*>(&m), 0, sizeof(m));
    st = fill_dist_params(dists[i], dt, m.a.d, dev);
    if (st != SDR_OK) return st;
    if (cv.numel == 0) continue;
    if (outs[i] == nullptr) return SDR_E_INVALID;
    m.a.g = make_gen(rngs[i]);
    m.a.ix = make_indexer(cv);
    m.a.out = outs[i];
    const bool fast = cv.istride == 1 && cv.inner % kV == 0 && aligned16(outs[i]);
    setup_chunks(cv, fast, m.a.nchunks, m.a.chunks_per_row, m.a.div_cpr);
    m.a.aligned = fast && chunks_aligned(cv, rngs[i].theta, kV);
    m.tiles = (static_cast<uint64_t>(cv.numel) + kTileElems - 1) / kTileElems;
    groups[dists[i].kind * 8 + dt].push_back(m);
  }
  for (int gi = 0; gi < static_cast<int>(groups.size()); ++gi) {
    auto& G = groups[gi];
    if (G.empty()) continue;
    const int kind = gi / 8, dt = gi % 8, m = static_cast<int>(G.size());
    FillArgs* d_descs = nullptr;
    uint64_t* d_prefix = nullptr;
    cudaError_t e = cudaMallocAsync(&d_descs, sizeof(FillArgs) * m, s);
    if (e == cudaSuccess) e = cudaMallocAsync(&d_prefix, sizeof(uint64_t) * (m + 1), s);  // + tile counter
    if (e != cudaSuccess) {
      set_cuda_error(e);
      return SDR_E_CUDA;
    }
    uint64_t tiles = 0;
    for (int i0 = 0; i0 < m; i0 += kUploadN) {
      auto U = std::make_unique<UploadArgs>();
      U->n = std::min(kUploadN, m - i0);
      U->dst = d_descs + i0;
      U->dst_prefix = d_prefix + i0;
      U->counter = i0 == 0 ? d_prefix + m : nullptr;
      for (int i = 0; i < U->n; ++i) {
        U->a[i] = G[i0 + i].a;
        U->prefix[i] = tiles;
        tiles += G[i0 + i].tiles;
      }
      k_upload_descs<<<1, 256, 0, s>>>(*U);
    }
    int st = with_dist(kind, [&](auto D) {
      constexpr int DIST = decltype(D)::value;
      return with_dtype<DIST>(dt, [&](auto T) {
        launch_batch<DIST, decltype(T)::value>(d_descs, d_prefix, m, tiles, s);
        return check_launch();
      });
    });
    cudaFreeAsync(d_descs, s);
    cudaFreeAsync(d_prefix, s);
    if (st != SDR_OK) return st;
  }
  return SDR_OK;
}

const char* last_cuda_error() { return g_cuda_err; }

}  // namespace sdr
