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
// a call run in one launch: CTAs walk a global tile list (binary search on the
// job prefix) and move 16 B vectors when the job is 16 B aligned.
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
  int64_t tiles;        // tiles of kTileBytes covering nspans*span_bytes
  int32_t vec;          // 16, 8, 4 or 1: widest aligned access
  int32_t pad_;
};

constexpr int64_t kTileBytes = 32768;

// Tiles never cross a span: tile t of a job is part (t % tiles_per_span) of
// span (t / tiles_per_span), so the inner loop is a plain strided vector copy.
template <typename V>
__device__ __forceinline__ void copy_part(const unsigned char* __restrict__ src,
                                          unsigned char* __restrict__ dst, int64_t nbytes) {
  const int64_t n = nbytes / static_cast<int64_t>(sizeof(V));
  const V* s = reinterpret_cast<const V*>(src);
  V* d = reinterpret_cast<V*>(dst);
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) d[i] = s[i];
}

__global__ void __launch_bounds__(256) k_copy_jobs(const CopyJob* __restrict__ jobs,
                                                   const int64_t* __restrict__ prefix, int n,
                                                   int64_t ntiles) {
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    int lo = 0, hi = n - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (prefix[mid] <= t) lo = mid;
      else hi = mid - 1;
    }
    const CopyJob& J = jobs[lo];
    const int64_t tps = (J.span_bytes + kTileBytes - 1) / kTileBytes;  // tiles per span
    const int64_t lt = t - prefix[lo];
    const int64_t span = lt / tps, part = lt - span * tps;
    const int64_t off = part * kTileBytes;
    const int64_t len = min(kTileBytes, J.span_bytes - off);
    const unsigned char* src = J.src + span * J.src_stride + off;
    unsigned char* dst = J.dst + span * J.dst_stride + off;
    switch (J.vec) {
      case 16: copy_part<uint4>(src, dst, len); break;
      case 8: copy_part<uint2>(src, dst, len); break;
      case 4: copy_part<uint32_t>(src, dst, len); break;
      default: copy_part<unsigned char>(src, dst, len); break;
    }
  }
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
  J.tiles = nspans * ((span_bytes + kTileBytes - 1) / kTileBytes);
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
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t cap = static_cast<int64_t>(sms) * 8;
  const int grid = static_cast<int>(tiles < cap ? tiles : cap);
  k_copy_jobs<<<grid, 256, 0, s>>>(d_jobs, d_prefix, n, tiles);
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
