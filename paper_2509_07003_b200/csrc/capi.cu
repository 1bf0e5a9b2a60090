// capi.cu -- the extern "C" boundary declared in include/sdrng.h.
#include "sdr_core.cuh"

namespace sdr {
int fill(void* out, int dt, const sdr_dist& dist, const sdr_rng& rng, const sdr_view& view,
         cudaStream_t s);
int fill_batch(void* const* outs, const int32_t* dts, const sdr_dist* dists, const sdr_rng* rngs,
               const sdr_view* views, int n, cudaStream_t s);
int dropout(const void* x, int xt, void* y, int yt, void* mask, int mt, double p,
            const sdr_rng& rng, const sdr_view& view, cudaStream_t s);
int transform(const uint32_t* w0, const uint32_t* w1, int64_t n, const sdr_dist& dist, void* out,
              int dt, cudaStream_t s);
int philox_blocks(const uint64_t* tau, const uint64_t* beta, int64_t n, uint64_t seed,
                  uint32_t* words, cudaStream_t s);
int normal_tables_load(int device, const double* r_host, const double* c_host, double* er,
                       double* ec);
int normal_tables_loaded(int device);
int normal_mirror_info(int device, uint64_t* device_bytes, uint64_t* exceptions, int32_t* compact,
                       double* build_ms);
int normal_delta_info(int device, uint64_t* device_bytes, uint64_t* escapes_r, uint64_t* escapes_c,
                      uint64_t* max_abs_r, uint64_t* max_abs_c);
int normal_fallback_count(int device, uint64_t* count);
int probe_int32(int device, double* imad_per_s, double* lop3_per_s, double* philox_per_s);
const char* last_cuda_error();
int unpack_gathered(const sdr_pack_member* m, int n, const void* packed, int64_t seg_bytes,
                    int nranks, cudaStream_t s);
int pack_scatter(const sdr_pack_member* m, int n, void* packed, int64_t seg_bytes, int nranks,
                 cudaStream_t s);
int pack_local(const sdr_pack_member* m, int n, void* seg, cudaStream_t s);
int unpack_local(const sdr_pack_member* m, int n, const void* seg, cudaStream_t s);
int slice_local(const sdr_pack_member* full, const sdr_pack_member* piece, int n, int rank, int nranks,
                cudaStream_t s);
int unpack_gathered_peers(const sdr_pack_member* m, int n, const void* const* segs, int nranks,
                          cudaStream_t s);
int reduce_scatter_peers(const sdr_pack_member* m, int n, const void* const* packed,
                         int64_t seg_bytes, int nranks, int rank, int dtype, cudaStream_t s);
int peer_barrier(void* const* flags, int rank, int nranks, uint64_t epoch, int64_t timeout_ns,
                 cudaStream_t s);
int peer_flag_read(const void* base, int index, uint64_t* value);
int peer_heap_alloc(int device, int64_t bytes, void** base, sdr_ipc_handle* handle);
int peer_heap_open(int device, const sdr_ipc_handle* handle, void** base);
int peer_heap_close(void* base);
int peer_heap_free(void* base);
}  // namespace sdr

static cudaStream_t as_stream(void* s) { return static_cast<cudaStream_t>(s); }

extern "C" {

int32_t sdr_version(void) { return 1; }

const char* sdr_strerror(int32_t status) {
  switch (status) {
    case SDR_OK: return "ok";
    case SDR_E_INVALID: return "invalid argument (shape, window, pointer or count)";
    case SDR_E_DTYPE: return "dtype not supported for this distribution/op";
    case SDR_E_DIST: return "unknown distribution kind";
    case SDR_E_PARAM: return "distribution parameter out of domain";
    case SDR_E_CUDA: return "CUDA error";
    case SDR_E_NOTABLES: return "normal() needs sdr_normal_tables_load on this device first";
    case SDR_E_ALIGN: return "buffer misaligned";
    default: return "unknown status";
  }
}

const char* sdr_last_cuda_error(void) { return sdr::last_cuda_error(); }

int32_t sdr_philox_block_host(uint64_t seed, uint64_t tau, uint64_t beta, uint32_t out[4]) {
  if (out == nullptr) return SDR_E_INVALID;
  sdr::philox10(seed, tau, beta, out);
  return SDR_OK;
}

int32_t sdr_philox_blocks(const uint64_t* tau, const uint64_t* beta, int64_t n, uint64_t seed,
                          uint32_t* words, void* stream) {
  return sdr::philox_blocks(tau, beta, n, seed, words, as_stream(stream));
}

int32_t sdr_fill(void* out, int32_t out_dtype, const sdr_dist* dist, const sdr_rng* rng,
                 const sdr_view* view, void* stream) {
  if (dist == nullptr || rng == nullptr || view == nullptr) return SDR_E_INVALID;
  return sdr::fill(out, out_dtype, *dist, *rng, *view, as_stream(stream));
}

int32_t sdr_transform(const uint32_t* w0, const uint32_t* w1, int64_t n, const sdr_dist* dist,
                      void* out, int32_t out_dtype, void* stream) {
  if (dist == nullptr) return SDR_E_INVALID;
  return sdr::transform(w0, w1, n, *dist, out, out_dtype, as_stream(stream));
}

int32_t sdr_fill_batch(void* const* outs, const int32_t* out_dtypes, const sdr_dist* dists,
                       const sdr_rng* rngs, const sdr_view* views, int32_t n, void* stream) {
  return sdr::fill_batch(outs, out_dtypes, dists, rngs, views, n, as_stream(stream));
}

int32_t sdr_dropout(const void* x, int32_t x_dtype, void* y, int32_t y_dtype, void* mask,
                    int32_t mask_dtype, double p, const sdr_rng* rng, const sdr_view* view,
                    void* stream) {
  if (rng == nullptr || view == nullptr) return SDR_E_INVALID;
  return sdr::dropout(x, x_dtype, y, y_dtype, mask, mask_dtype, p, *rng, *view, as_stream(stream));
}

int32_t sdr_normal_tables_load(int32_t device, const double* log1p_table, const double* c_table,
                               double* max_rel_err_r, double* max_abs_err_c) {
  return sdr::normal_tables_load(device, log1p_table, c_table, max_rel_err_r, max_abs_err_c);
}

int32_t sdr_normal_tables_loaded(int32_t device) { return sdr::normal_tables_loaded(device); }

int32_t sdr_normal_mirror_info(int32_t device, uint64_t* device_bytes, uint64_t* exceptions,
                               int32_t* compact, double* build_ms) {
  return sdr::normal_mirror_info(device, device_bytes, exceptions, compact, build_ms);
}

int32_t sdr_normal_delta_info(int32_t device, uint64_t* device_bytes, uint64_t* escapes_r, uint64_t* escapes_c,
                              uint64_t* max_abs_r, uint64_t* max_abs_c) {
  return sdr::normal_delta_info(device, device_bytes, escapes_r, escapes_c, max_abs_r, max_abs_c);
}
int32_t sdr_normal_fallback_count(int32_t device, uint64_t* count) {
  return sdr::normal_fallback_count(device, count);
}

int32_t sdr_unpack_gathered(const sdr_pack_member* members, int32_t n, const void* packed,
                            int64_t seg_bytes, int32_t nranks, void* stream) {
  return sdr::unpack_gathered(members, n, packed, seg_bytes, nranks, as_stream(stream));
}

int32_t sdr_pack_scatter(const sdr_pack_member* members, int32_t n, void* packed,
                         int64_t seg_bytes, int32_t nranks, void* stream) {
  return sdr::pack_scatter(members, n, packed, seg_bytes, nranks, as_stream(stream));
}

int32_t sdr_pack_local(const sdr_pack_member* members, int32_t n, void* segment, void* stream) {
  return sdr::pack_local(members, n, segment, as_stream(stream));
}

int32_t sdr_unpack_local(const sdr_pack_member* members, int32_t n, const void* segment,
                         void* stream) {
  return sdr::unpack_local(members, n, segment, as_stream(stream));
}

int32_t sdr_slice_local(const sdr_pack_member* full, const sdr_pack_member* piece, int32_t n,
                        int32_t rank, int32_t nranks, void* stream) {
  return sdr::slice_local(full, piece, n, rank, nranks, as_stream(stream));
}

int32_t sdr_peer_heap_alloc(int32_t device, int64_t bytes, void** base, sdr_ipc_handle* handle) {
  return sdr::peer_heap_alloc(device, bytes, base, handle);
}

int32_t sdr_peer_heap_open(int32_t device, const sdr_ipc_handle* handle, void** base) {
  return sdr::peer_heap_open(device, handle, base);
}

int32_t sdr_peer_heap_close(void* base) { return sdr::peer_heap_close(base); }

int32_t sdr_peer_heap_free(void* base) { return sdr::peer_heap_free(base); }

int32_t sdr_peer_barrier(void* const* flags, int32_t rank, int32_t nranks, uint64_t epoch,
                         int64_t timeout_ns, void* stream) {
  return sdr::peer_barrier(flags, rank, nranks, epoch, timeout_ns, as_stream(stream));
}

int32_t sdr_peer_flag_read(const void* base, int32_t index, uint64_t* value) {
  return sdr::peer_flag_read(base, index, value);
}

int32_t sdr_unpack_gathered_peers(const sdr_pack_member* members, int32_t n,
                                  const void* const* segs, int32_t nranks, void* stream) {
  return sdr::unpack_gathered_peers(members, n, segs, nranks, as_stream(stream));
}

int32_t sdr_reduce_scatter_peers(const sdr_pack_member* members, int32_t n,
                                 const void* const* packed, int64_t seg_bytes, int32_t nranks,
                                 int32_t rank, int32_t dtype, void* stream) {
  return sdr::reduce_scatter_peers(members, n, packed, seg_bytes, nranks, rank, dtype,
                                   as_stream(stream));
}

int32_t sdr_peer_all_gather(const sdr_pack_member* send, const sdr_pack_member* recv, int32_t n,
                            void* const* bases, int32_t nranks, int32_t rank, int64_t half_offset,
                            uint64_t epoch, int64_t timeout_ns, int32_t lead_barrier, void* stream) {
  if (bases == nullptr || nranks < 1 || nranks > SDR_MAX_PEERS || rank < 0 || rank >= nranks || half_offset < 0)
    return SDR_E_INVALID;
  const void* segs[SDR_MAX_PEERS];
  for (int q = 0; q < nranks; ++q) segs[q] = static_cast<const char*>(bases[q]) + half_offset;
  const cudaStream_t s = as_stream(stream);
  int st = SDR_OK;
  if (lead_barrier) {
    st = sdr::peer_barrier(bases, rank, nranks, epoch, timeout_ns, s);
    if (epoch != 0) ++epoch;
  }
  if (st == SDR_OK) st = sdr::pack_local(send, n, const_cast<void*>(segs[rank]), s);
  if (st == SDR_OK) st = sdr::peer_barrier(bases, rank, nranks, epoch, timeout_ns, s);
  if (st == SDR_OK) st = sdr::unpack_gathered_peers(recv, n, segs, nranks, s);
  return st;
}

int32_t sdr_peer_reduce_scatter(const sdr_pack_member* full, const sdr_pack_member* piece, int32_t n,
                                void* const* bases, int32_t nranks, int32_t rank, int64_t half_offset,
                                int64_t seg_bytes, int32_t dtype, uint64_t epoch, int64_t timeout_ns,
                                int32_t lead_barrier, void* stream) {
  if (bases == nullptr || nranks < 1 || nranks > SDR_MAX_PEERS || rank < 0 || rank >= nranks || half_offset < 0)
    return SDR_E_INVALID;
  const void* segs[SDR_MAX_PEERS];
  for (int q = 0; q < nranks; ++q) segs[q] = static_cast<const char*>(bases[q]) + half_offset;
  const cudaStream_t s = as_stream(stream);
  int st = SDR_OK;
  if (lead_barrier) {
    st = sdr::peer_barrier(bases, rank, nranks, epoch, timeout_ns, s);
    if (epoch != 0) ++epoch;
  }
  if (st == SDR_OK) st = sdr::pack_scatter(full, n, const_cast<void*>(segs[rank]), seg_bytes, nranks, s);
  if (st == SDR_OK) st = sdr::peer_barrier(bases, rank, nranks, epoch, timeout_ns, s);
  if (st == SDR_OK) st = sdr::reduce_scatter_peers(piece, n, segs, seg_bytes, nranks, rank, dtype, s);
  return st;
}

int32_t sdr_probe_int32(int32_t device, double* imad_wide_per_s, double* lop3_per_s,
                        double* philox_blocks_per_s) {
  return sdr::probe_int32(device, imad_wide_per_s, lop3_per_s, philox_blocks_per_s);
}

}  // extern "C"
