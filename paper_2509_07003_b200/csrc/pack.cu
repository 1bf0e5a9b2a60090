// pack.cu -- multi-DTensor pack / unpack around ONE coalesced NCCL collective.
//
// Replaces the reference's per-fiber Python copies: the np.concatenate packing
// of comm.py:189-192 / 269-272, the unpack loops of comm.py:194-199 / 274-279,
// _assemble_shards (dtensor.py:261-283) and _local_slice (dtensor.py:286-298).
//
// Every member tensor is viewed as [outer, rows, inner] around the tensor dim
// being gathered / scattered; a rank's piece along `rows` is the ceil-block
// [r*chunk, min((r+1)*chunk, rows)) (placement.py:226-231), padded to `chunk`
// rows in the packed buffer so NCCL sees equal-size rank segments.  For fixed
// `outer` index both the tensor piece and its slot are one contiguous byte
// span, so each (member, rank) pair is a batched 2-D copy ("job").  All jobs of
// a call run in one launch with one CTA per tile (binary search on the job
// prefix), moving 16 B vectors when every job is 16 B aligned.
#include <cstring>
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

template <typename V>
__device__ __forceinline__ void copy_tile(const CopyJob* __restrict__ jobs,
                                          const int64_t* __restrict__ prefix, int n) {
  constexpr int U = static_cast<int>(kTileBytes / (sizeof(V) * 256));
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
    off = (lt - s0 * J.parts) * kTileBytes;
    len = min(kTileBytes, J.span_bytes - off);
  }
  const int lv = static_cast<int>(len / static_cast<int64_t>(sizeof(V)));
  const int total = cnt * lv;
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
  const V* sv[U];
  V* dv[U];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    sv[u] = reinterpret_cast<const V*>(sp);
    dv[u] = reinterpret_cast<V*>(dp);
    sp += s_step;
    dp += d_step;
    c += dc;
    if (c >= lv) {
      c -= lv;
      sp += s_wrap;
      dp += d_wrap;
    }
  }
  V v[U];
#pragma unroll
  for (int u = 0; u < U; ++u)
    if (static_cast<int>(threadIdx.x) + u * 256 < total) v[u] = *sv[u];
#pragma unroll
  for (int u = 0; u < U; ++u)
    if (static_cast<int>(threadIdx.x) + u * 256 < total) *dv[u] = v[u];
}

// Job table in device memory (large calls).
template <typename V>
__global__ void __launch_bounds__(256) k_copy_tiles(const CopyJob* __restrict__ jobs,
                                                    const int64_t* __restrict__ prefix, int n) {
  copy_tile<V>(jobs, prefix, n);
}

// Small calls (the common case: a layer's members x ranks): the job table is a
// kernel parameter -- no allocation or H2D copy per call, and the launch is
// stream-capturable into a CUDA graph.
constexpr int kParamJobs = 96;
struct JobTable {
  int32_t n;
  int32_t pad_;
  int64_t prefix[kParamJobs];
  CopyJob jobs[kParamJobs];
};

template <typename V>
__global__ void __launch_bounds__(256) k_copy_tiles_p(const __grid_constant__ JobTable T) {
  copy_tile<V>(T.jobs, T.prefix, T.n);
}

static int widest(std::initializer_list<int64_t> vals) {
  int64_t acc = 0;
  for (int64_t v : vals) acc |= v;
  if ((acc & 15) == 0) return 16;
  if ((acc & 7) == 0) return 8;
  if ((acc & 3) == 0) return 4;
  return 1;
}

static void add_job(std::vector<CopyJob>& jobs, const void* src, void* dst, int64_t nspans,
                    int64_t span_bytes, int64_t src_stride, int64_t dst_stride) {
  if (nspans <= 0 || span_bytes <= 0) return;
  CopyJob J;
  memset(&J, 0, sizeof(J));
  J.src = static_cast<const unsigned char*>(src);
  J.dst = static_cast<unsigned char*>(dst);
  J.nspans = nspans;
  J.span_bytes = span_bytes;
  J.src_stride = src_stride;
  J.dst_stride = dst_stride;
  if (span_bytes < kTileBytes) {
    J.spt = kTileBytes / span_bytes;
    J.parts = 1;
    J.tiles = (nspans + J.spt - 1) / J.spt;
  } else {
    J.spt = 1;
    J.parts = (span_bytes + kTileBytes - 1) / kTileBytes;
    J.tiles = nspans * J.parts;
  }
  J.vec = widest({static_cast<int64_t>(reinterpret_cast<uintptr_t>(src)),
                  static_cast<int64_t>(reinterpret_cast<uintptr_t>(dst)), span_bytes, src_stride,
                  dst_stride});
  jobs.push_back(J);
}

static int run_jobs(const std::vector<CopyJob>& jobs, cudaStream_t s) {
  if (jobs.empty()) return SDR_OK;
  const int n = static_cast<int>(jobs.size());
  std::vector<int64_t> prefix(n);
  int64_t tiles = 0;
  for (int i = 0; i < n; ++i) {
    prefix[i] = tiles;
    tiles += jobs[i].tiles;
  }
  // vector width of the whole call: the narrowest job's (jobs are few and large)
  int vec = 16;
  for (const CopyJob& J : jobs) vec = J.vec < vec ? J.vec : vec;
  const unsigned grid = static_cast<unsigned>(tiles);
  if (n <= kParamJobs) {
    JobTable T;
    memset(static_cast<void*>(&T), 0, sizeof(T));
    T.n = n;
    for (int i = 0; i < n; ++i) {
      T.prefix[i] = prefix[i];
      T.jobs[i] = jobs[i];
    }
    switch (vec) {
      case 16: k_copy_tiles_p<uint4><<<grid, 256, 0, s>>>(T); break;
      case 8: k_copy_tiles_p<uint2><<<grid, 256, 0, s>>>(T); break;
      case 4: k_copy_tiles_p<uint32_t><<<grid, 256, 0, s>>>(T); break;
      default: k_copy_tiles_p<unsigned char><<<grid, 256, 0, s>>>(T); break;
    }
    return check_launch();
  }
  CopyJob* d_jobs = nullptr;
  int64_t* d_prefix = nullptr;
  cudaError_t e = cudaMallocAsync(&d_jobs, sizeof(CopyJob) * n, s);
  if (e == cudaSuccess) e = cudaMallocAsync(&d_prefix, sizeof(int64_t) * n, s);
  if (e == cudaSuccess) e = cudaMemcpyAsync(d_jobs, jobs.data(), sizeof(CopyJob) * n, cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess) e = cudaMemcpyAsync(d_prefix, prefix.data(), sizeof(int64_t) * n, cudaMemcpyHostToDevice, s);
  if (e != cudaSuccess) {
    set_cuda_error(e);
    return SDR_E_CUDA;
  }
  switch (vec) {
    case 16: k_copy_tiles<uint4><<<grid, 256, 0, s>>>(d_jobs, d_prefix, n); break;
    case 8: k_copy_tiles<uint2><<<grid, 256, 0, s>>>(d_jobs, d_prefix, n); break;
    case 4: k_copy_tiles<uint32_t><<<grid, 256, 0, s>>>(d_jobs, d_prefix, n); break;
    default: k_copy_tiles<unsigned char><<<grid, 256, 0, s>>>(d_jobs, d_prefix, n); break;
  }
  const int st = check_launch();
  cudaFreeAsync(d_jobs, s);
  cudaFreeAsync(d_prefix, s);
  return st;
}

static bool member_ok(const sdr_pack_member& m) {
  return m.outer >= 0 && m.rows >= 0 && m.inner >= 0 && m.chunk_rows >= 0 && m.seg_off >= 0 &&
         (m.elem_bytes == 1 || m.elem_bytes == 2 || m.elem_bytes == 4 || m.elem_bytes == 8);
}

// Rank r's row range of a `rows`-long dim split in chunks of `chunk`.
static void rank_rows(int64_t rows, int64_t chunk, int r, int64_t& lo, int64_t& len) {
  lo = static_cast<int64_t>(r) * chunk;
  if (lo > rows) lo = rows;
  int64_t hi = lo + chunk;
  if (hi > rows) hi = rows;
  len = hi - lo;
}

int unpack_gathered(const sdr_pack_member* M, int n, const void* packed, int64_t seg_bytes,
                    int nranks, cudaStream_t s) {
  if (n < 0 || nranks < 1 || seg_bytes < 0 || (n > 0 && (M == nullptr || packed == nullptr)))
    return SDR_E_INVALID;
  std::vector<CopyJob> jobs;
  for (int i = 0; i < n; ++i) {
    const sdr_pack_member& m = M[i];
    if (!member_ok(m) || m.chunk_rows * nranks < m.rows) return SDR_E_INVALID;
    const int64_t eb = m.elem_bytes, row_b = m.inner * eb;
    if (m.seg_off + m.outer * m.chunk_rows * row_b > seg_bytes) return SDR_E_INVALID;
    for (int r = 0; r < nranks; ++r) {
      int64_t lo, len;
      rank_rows(m.rows, m.chunk_rows, r, lo, len);
      const unsigned char* src = static_cast<const unsigned char*>(packed) + r * seg_bytes + m.seg_off;
      unsigned char* dst = static_cast<unsigned char*>(m.data) + lo * row_b;
      add_job(jobs, src, dst, m.outer, len * row_b, m.chunk_rows * row_b, m.rows * row_b);
    }
  }
  return run_jobs(jobs, s);
}

int pack_scatter(const sdr_pack_member* M, int n, void* packed, int64_t seg_bytes, int nranks,
                 cudaStream_t s) {
  if (n < 0 || nranks < 1 || seg_bytes < 0 || (n > 0 && (M == nullptr || packed == nullptr)))
    return SDR_E_INVALID;
  std::vector<CopyJob> jobs;
  for (int i = 0; i < n; ++i) {
    const sdr_pack_member& m = M[i];
    if (!member_ok(m) || m.chunk_rows * nranks < m.rows) return SDR_E_INVALID;
    const int64_t eb = m.elem_bytes, row_b = m.inner * eb;
    if (m.seg_off + m.outer * m.chunk_rows * row_b > seg_bytes) return SDR_E_INVALID;
    for (int r = 0; r < nranks; ++r) {
      int64_t lo, len;
      rank_rows(m.rows, m.chunk_rows, r, lo, len);
      const unsigned char* src = static_cast<const unsigned char*>(m.data) + lo * row_b;
      unsigned char* dst = static_cast<unsigned char*>(packed) + r * seg_bytes + m.seg_off;
      add_job(jobs, src, dst, m.outer, len * row_b, m.rows * row_b, m.chunk_rows * row_b);
    }
  }
  return run_jobs(jobs, s);
}

int pack_local(const sdr_pack_member* M, int n, void* seg, cudaStream_t s) {
  if (n < 0 || (n > 0 && (M == nullptr || seg == nullptr))) return SDR_E_INVALID;
  std::vector<CopyJob> jobs;
  for (int i = 0; i < n; ++i) {
    const sdr_pack_member& m = M[i];
    if (!member_ok(m) || m.rows > m.chunk_rows) return SDR_E_INVALID;
    const int64_t row_b = m.inner * m.elem_bytes;
    add_job(jobs, m.data, static_cast<unsigned char*>(seg) + m.seg_off, m.outer, m.rows * row_b,
            m.rows * row_b, m.chunk_rows * row_b);
  }
  return run_jobs(jobs, s);
}

int unpack_local(const sdr_pack_member* M, int n, const void* seg, cudaStream_t s) {
  if (n < 0 || (n > 0 && (M == nullptr || seg == nullptr))) return SDR_E_INVALID;
  std::vector<CopyJob> jobs;
  for (int i = 0; i < n; ++i) {
    const sdr_pack_member& m = M[i];
    if (!member_ok(m) || m.rows > m.chunk_rows) return SDR_E_INVALID;
    const int64_t row_b = m.inner * m.elem_bytes;
    add_job(jobs, static_cast<const unsigned char*>(seg) + m.seg_off, m.data, m.outer,
            m.rows * row_b, m.chunk_rows * row_b, m.rows * row_b);
  }
  return run_jobs(jobs, s);
}

}  // namespace sdr
