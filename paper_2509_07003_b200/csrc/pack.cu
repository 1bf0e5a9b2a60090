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

#include "copy_tiles.cuh"

namespace sdr {

template <typename V>
__device__ __forceinline__ void copy_tile(const CopyJob* __restrict__ jobs,
                                          const int64_t* __restrict__ prefix, int n) {
  constexpr int U = static_cast<int>(kTileBytes / (sizeof(V) * 256));
  const unsigned char* sv[U];
  unsigned char* dv[U];
  const int total = tile_slots<V, U>(jobs, prefix, n, sv, dv);
  V v[U];
#pragma unroll
  for (int u = 0; u < U; ++u)
    if (static_cast<int>(threadIdx.x) + u * 256 < total) v[u] = *reinterpret_cast<const V*>(sv[u]);
#pragma unroll
  for (int u = 0; u < U; ++u)
    if (static_cast<int>(threadIdx.x) + u * 256 < total) *reinterpret_cast<V*>(dv[u]) = v[u];
}

// Job table in device memory (large calls).
template <typename V>
__global__ void __launch_bounds__(256) k_copy_tiles(const CopyJob* __restrict__ jobs,
                                                    const int64_t* __restrict__ prefix, int n) {
  copy_tile<V>(jobs, prefix, n);
}

// Small calls: the job table (JobTable, copy_tiles.cuh) is a kernel parameter.

template <typename V>
__global__ void __launch_bounds__(256) k_copy_tiles_p(const __grid_constant__ JobTable T) {
  copy_tile<V>(T.jobs, T.prefix, T.n);
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
      case 2: k_copy_tiles_p<uint16_t><<<grid, 256, 0, s>>>(T); break;
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
    case 2: k_copy_tiles<uint16_t><<<grid, 256, 0, s>>>(d_jobs, d_prefix, n); break;
    default: k_copy_tiles<unsigned char><<<grid, 256, 0, s>>>(d_jobs, d_prefix, n); break;
  }
  const int st = check_launch();
  cudaFreeAsync(d_jobs, s);
  cudaFreeAsync(d_prefix, s);
  return st;
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

// Replicate -> Shard local slice (dtensor.py:247-251, _local_slice
// dtensor.py:286-298): rank `rank`'s ceil-block rows of each full member into
// its piece tensor, one batched 2-D copy job per member.
int slice_local(const sdr_pack_member* F, const sdr_pack_member* Pc, int n, int rank, int nranks,
                cudaStream_t s) {
  if (n < 0 || nranks < 1 || rank < 0 || rank >= nranks || (n > 0 && (F == nullptr || Pc == nullptr)))
    return SDR_E_INVALID;
  std::vector<CopyJob> jobs;
  for (int i = 0; i < n; ++i) {
    const sdr_pack_member& f = F[i];
    const sdr_pack_member& p = Pc[i];
    if (!member_ok(f) || f.chunk_rows * nranks < f.rows) return SDR_E_INVALID;
    int64_t lo, len;
    rank_rows(f.rows, f.chunk_rows, rank, lo, len);
    if (p.outer != f.outer || p.inner != f.inner || p.elem_bytes != f.elem_bytes || p.rows != len)
      return SDR_E_INVALID;
    if (len == 0 || f.outer == 0 || f.inner == 0) continue;
    if (p.data == nullptr) return SDR_E_INVALID;
    const int64_t row_b = f.inner * f.elem_bytes;
    add_job(jobs, static_cast<const unsigned char*>(f.data) + lo * row_b, p.data, f.outer, len * row_b,
            f.rows * row_b, len * row_b);
  }
  return run_jobs(jobs, s);
}

// Force-load the copy kernels (CUDA lazy loading loads a kernel at its first
// launch, and that load waits for running kernels: a host thread that launches
// a not-yet-loaded kernel behind a spinning peer barrier would stall).
int preload_copy_kernels() {
  cudaFuncAttributes a;
  cudaError_t e = cudaSuccess;
  const void* fns[] = {
      reinterpret_cast<const void*>(&k_copy_tiles_p<uint4>), reinterpret_cast<const void*>(&k_copy_tiles_p<uint2>),
      reinterpret_cast<const void*>(&k_copy_tiles_p<uint32_t>), reinterpret_cast<const void*>(&k_copy_tiles_p<uint16_t>),
      reinterpret_cast<const void*>(&k_copy_tiles_p<unsigned char>), reinterpret_cast<const void*>(&k_copy_tiles<uint4>),
      reinterpret_cast<const void*>(&k_copy_tiles<uint2>), reinterpret_cast<const void*>(&k_copy_tiles<uint32_t>),
      reinterpret_cast<const void*>(&k_copy_tiles<uint16_t>), reinterpret_cast<const void*>(&k_copy_tiles<unsigned char>)};
  for (const void* f : fns)
    if (e == cudaSuccess) e = cudaFuncGetAttributes(&a, f);
  if (e != cudaSuccess) {
    set_cuda_error(e);
    return SDR_E_CUDA;
  }
  return SDR_OK;
}

}  // namespace sdr
