// copy_tiles.cuh -- the tiled multi-job copy geometry shared by the pack /
// unpack kernels (pack.cu) and the peer-memory collectives (peer.cu).
#pragma once

#include <cstring>
#include <initializer_list>
#include <vector>

#include "sdr_core.cuh"

namespace sdr {

struct CopyJob {
  const unsigned char* src;
  unsigned char* dst;
  int64_t nspans;       // number of spans (the `outer` extent)
  int64_t span_bytes;   // bytes per span
  int64_t src_stride;   // bytes between spans in src
  int64_t dst_stride;   // bytes between spans in dst
  int64_t tiles;        // tiles covering the job (see tile_geometry)
  int64_t spt;          // spans per tile (>= 1; > 1 only when a span is < kTileBytes)
  int64_t parts;        // tiles per span (>= 1; > 1 only when spt == 1)
  int32_t vec;          // 16, 8, 4 or 1: widest aligned access
  int32_t pad_;
};

// A tile is <= kTileBytes of one job: `spt` whole spans when spans are short
// (e.g. the 4 KiB half-rows of a Shard(1) bf16 [4096, 4096] weight), or one
// kTileBytes part of a long span.  One CTA per tile: 256 threads x U vectors,
// all loads issued before the stores; the CTA scheduler keeps a moving front
// of tiles in flight (measured: per-CTA tiles beat persistent grids and TMA
// bulk-copy variants on B200; 16 KiB tiles reach the torch-copy rate, 6.3 TB/s).
#ifndef SDR_COPY_TILE
#define SDR_COPY_TILE 16384
#endif
constexpr int64_t kTileBytes = SDR_COPY_TILE;

// Tile `blockIdx.x` of the call: the job (binary search on the prefix), then
// per thread the U (source, destination) addresses of its vectors; returns the
// number of valid vectors in the tile (thread t owns vectors t + 256u).
template <typename V, int U>
__device__ __forceinline__ int tile_slots(const CopyJob* __restrict__ jobs,
                                          const int64_t* __restrict__ prefix, int n,
                                          const unsigned char* (&sv)[U], unsigned char* (&dv)[U]) {
  // tile bytes = U vectors x 256 threads (jobs are built with the same size)
  constexpr int64_t kTB = static_cast<int64_t>(U) * sizeof(V) * 256;
  const int64_t t = blockIdx.x;
  int lo = 0, hi = n - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (prefix[mid] <= t) lo = mid;
    else hi = mid - 1;
  }
  const CopyJob& J = jobs[lo];
  const int64_t lt = t - prefix[lo];
  int64_t s0, off, len;
  int cnt;
  if (J.spt > 1) {
    s0 = lt * J.spt;
    cnt = static_cast<int>(min(J.spt, J.nspans - s0));
    off = 0;
    len = J.span_bytes;
  } else {
    s0 = lt / J.parts;
    cnt = 1;
    off = (lt - s0 * J.parts) * kTB;
    len = min(kTB, J.span_bytes - off);
  }
  const int lv = static_cast<int>(len / static_cast<int64_t>(sizeof(V)));
  // Thread element i = tid + 256u -> (span r, vector c), stepped incrementally:
  // one division per thread, then +256 = (dr spans, dc vectors) with a carry.
  const int dr = 256 / lv, dc = 256 - dr * lv;
  int r = threadIdx.x / lv, c = threadIdx.x - r * lv;
  const unsigned char* sp = J.src + (s0 + r) * J.src_stride + off + c * static_cast<int64_t>(sizeof(V));
  unsigned char* dp = J.dst + (s0 + r) * J.dst_stride + off + c * static_cast<int64_t>(sizeof(V));
  const int64_t s_step = dr * J.src_stride + dc * static_cast<int64_t>(sizeof(V));
  const int64_t d_step = dr * J.dst_stride + dc * static_cast<int64_t>(sizeof(V));
  const int64_t s_wrap = J.src_stride - lv * static_cast<int64_t>(sizeof(V));
  const int64_t d_wrap = J.dst_stride - lv * static_cast<int64_t>(sizeof(V));
#pragma unroll
  for (int u = 0; u < U; ++u) {
    sv[u] = sp;
    dv[u] = dp;
    sp += s_step;
    dp += d_step;
    c += dc;
    if (c >= lv) {
      c -= lv;
      sp += s_wrap;
      dp += d_wrap;
    }
  }
  return cnt * lv;
}


// Small calls (the common case: a layer's members x ranks): the job table is a
// kernel parameter -- no allocation or H2D copy per call, and the launch is
// stream-capturable into a CUDA graph.
#ifndef SDR_PARAM_JOBS
#define SDR_PARAM_JOBS 96
#endif
constexpr int kParamJobs = SDR_PARAM_JOBS;
struct JobTable {
  int32_t n;
  int32_t pad_;
  int64_t prefix[kParamJobs];
  CopyJob jobs[kParamJobs];
};

inline int widest(std::initializer_list<int64_t> vals) {
  int64_t acc = 0;
  for (int64_t v : vals) acc |= v;
  if ((acc & 15) == 0) return 16;
  if ((acc & 7) == 0) return 8;
  if ((acc & 3) == 0) return 4;
  if ((acc & 1) == 0) return 2;
  return 1;
}

inline void add_job(std::vector<CopyJob>& jobs, const void* src, void* dst, int64_t nspans,
                    int64_t span_bytes, int64_t src_stride, int64_t dst_stride,
                    int64_t tile_bytes = kTileBytes) {
  if (nspans <= 0 || span_bytes <= 0) return;
  CopyJob J;
  memset(&J, 0, sizeof(J));
  J.src = static_cast<const unsigned char*>(src);
  J.dst = static_cast<unsigned char*>(dst);
  J.nspans = nspans;
  J.span_bytes = span_bytes;
  J.src_stride = src_stride;
  J.dst_stride = dst_stride;
  if (span_bytes < tile_bytes) {
    J.spt = tile_bytes / span_bytes;
    J.parts = 1;
    J.tiles = (nspans + J.spt - 1) / J.spt;
  } else {
    J.spt = 1;
    J.parts = (span_bytes + tile_bytes - 1) / tile_bytes;
    J.tiles = nspans * J.parts;
  }
  J.vec = widest({static_cast<int64_t>(reinterpret_cast<uintptr_t>(src)),
                  static_cast<int64_t>(reinterpret_cast<uintptr_t>(dst)), span_bytes, src_stride,
                  dst_stride});
  jobs.push_back(J);
}

inline bool member_ok(const sdr_pack_member& m) {
  return m.outer >= 0 && m.rows >= 0 && m.inner >= 0 && m.chunk_rows >= 0 && m.seg_off >= 0 &&
         (m.elem_bytes == 1 || m.elem_bytes == 2 || m.elem_bytes == 4 || m.elem_bytes == 8);
}

// Rank r's row range of a `rows`-long dim split in chunks of `chunk`.
inline void rank_rows(int64_t rows, int64_t chunk, int r, int64_t& lo, int64_t& len) {
  lo = static_cast<int64_t>(r) * chunk;
  if (lo > rows) lo = rows;
  int64_t hi = lo + chunk;
  if (hi > rows) hi = rows;
  len = hi - lo;
}

}  // namespace sdr
