/* sdrng.h -- C ABI of the B200-native single-device-semantic distributed RNG
 * and the multi-DTensor pack/unpack used by the fused redistribute.
 *
 * The reference (veScale spmdsim, /root/reference/pkg/src/spmdsim) is pure
 * Python/NumPy and has no FFI; its boundary for this path is the Python API of
 * spmdsim.rng / placement / dtensor / comm.  Each entry point below replaces
 * one reference function (cited), and the Python package
 * paper_2509_07003_b200 binds them with ctypes.
 *
 * Conventions
 *  - Every call is asynchronous on `stream` (a cudaStream_t passed as void*;
 *    NULL = legacy default stream) and returns an sdr_status (0 = OK).
 *  - The caller owns every buffer.  Device buffers are plain device pointers.
 *  - The library holds no RNG state: (seed, offset, theta) are passed by value
 *    and advanced by the caller exactly as rng.py:95-98.
 *  - The fill and dropout fast kernels use programmatic dependent launch: a
 *    following PDL launch may start its CTAs while ours drain, and every one of
 *    our kernels executes griddepcontrol.wait before touching memory a previous
 *    grid may use, so stream order is preserved for all data.  Launches are
 *    CUDA-graph capturable (the pack/unpack job table of calls with <= 96 jobs
 *    is a kernel parameter; larger calls stage it with cudaMallocAsync).
 *  - A window ("view") of a row-major global tensor of rank `ndim` is given per
 *    tensor dim d by global_shape[d], local_start[d], local_len[d], and for
 *    InterleavedShard dims groups[d] (m) and group_stride[d] (global distance
 *    between groups); groups == NULL means every dim is contiguous.  Local
 *    element order is row-major over local_len (placement.py:202-223).
 */
#ifndef SDRNG_H_
#define SDRNG_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SDR_MAX_NDIM 8

typedef enum {
  SDR_OK = 0,
  SDR_E_INVALID = 1,     /* bad shape / window / pointer / count            */
  SDR_E_DTYPE = 2,       /* dtype unsupported for this distribution/op      */
  SDR_E_DIST = 3,        /* unknown distribution kind                       */
  SDR_E_PARAM = 4,       /* distribution parameter out of domain (ValueError) */
  SDR_E_CUDA = 5,        /* CUDA launch/runtime error                       */
  SDR_E_NOTABLES = 6,    /* normal() before sdr_normal_tables_load          */
  SDR_E_ALIGN = 7        /* buffer misaligned for the requested op          */
} sdr_status;

typedef enum {
  SDR_F32 = 0, SDR_F64 = 1, SDR_BF16 = 2, SDR_F16 = 3,
  SDR_I64 = 4, SDR_I32 = 5, SDR_U8 = 6, SDR_BOOL = 7
} sdr_dtype;

typedef enum {
  SDR_UNIFORM01 = 0,  /* rng.py:118-127  */
  SDR_UNIFORM = 1,    /* rng.py:130-138  fparam = {lo, hi}      */
  SDR_NORMAL = 2,     /* rng.py:141-156  fparam = {mean, std}   */
  SDR_RANDINT = 3,    /* rng.py:159-171  iparam = {lo, hi}      */
  SDR_BERNOULLI = 4   /* rng.py:174-182  fparam = {p}           */
} sdr_dist_kind;

typedef struct {
  int32_t kind;        /* sdr_dist_kind */
  double fparam[2];
  int64_t iparam[2];
} sdr_dist;

typedef struct {        /* generator state, by value (rng.py:85-101) */
  uint64_t seed;
  uint64_t offset;
  uint64_t theta;       /* global_threads, >= 1 */
} sdr_rng;

typedef struct {        /* one window of a row-major global tensor */
  int32_t ndim;
  int64_t global_shape[SDR_MAX_NDIM];
  int64_t local_start[SDR_MAX_NDIM];
  int64_t local_len[SDR_MAX_NDIM];
  int64_t groups[SDR_MAX_NDIM];        /* 1 = contiguous; m for IS(d, m)       */
  int64_t group_stride[SDR_MAX_NDIM];  /* global index distance between groups */
} sdr_view;

/* Library identity / errors. */
int32_t sdr_version(void);
const char* sdr_strerror(int32_t status);
/* Last CUDA error string recorded by a failing call on this thread. */
const char* sdr_last_cuda_error(void);

/* Philox4x32-10 of one (seed, tau, beta) on the host: the same __host__
 * __device__ round function the kernels use.  Replaces backend_block
 * (rng.py:62-73).  out[4] = the four output words. */
int32_t sdr_philox_block_host(uint64_t seed, uint64_t tau, uint64_t beta, uint32_t out[4]);

/* Device Philox words for n (tau, beta) pairs (device arrays), writing
 * words[4*i + w].  Replaces philox_4x32_10 over arrays (rng.py:34-59). */
int32_t sdr_philox_blocks(const uint64_t* tau, const uint64_t* beta, int64_t n, uint64_t seed,
                          uint32_t* words, void* stream);

/* Fill one window: fill_random (rng.py:185-205) with any distribution
 * transform (rng.py:113-182).  `out` is the contiguous local tensor. */
int32_t sdr_fill(void* out, int32_t out_dtype, const sdr_dist* dist, const sdr_rng* rng,
                 const sdr_view* view, void* stream);

/* The distribution plug-in point Distribution.transform(words, dtype)
 * (rng.py:104-110; the five transforms rng.py:113-182): out[i] = value of
 * `dist` for the Philox block whose words 0 and 1 are w0[i], w1[i] (device
 * arrays of n uint32; no distribution reads words 2-3).  Same arithmetic as
 * sdr_fill (the fill kernels call the same device transform), so
 * transform(blocks(...)) == fill_random(...) bit for bit. */
int32_t sdr_transform(const uint32_t* w0, const uint32_t* w1, int64_t n, const sdr_dist* dist,
                      void* out, int32_t out_dtype, void* stream);

/* Multi-tensor fill: n independent fills in ONE launch per (distribution,
 * dtype) group (Module.materialize, model.py:121-132 -> generate_distributed,
 * rng.py:220-235).  Each fill has its own dist/rng/view/dtype -- every dtype
 * sdr_fill accepts for that distribution (float for all five, int64/int32
 * for RandInt, int/uint8/bool for Bernoulli).  Table arrays are host memory;
 * the descriptors reach the device as kernel parameters (no host copy), so
 * the call is stream-ordered end to end and may be captured in a CUDA graph. */
int32_t sdr_fill_batch(void* const* outs, const int32_t* out_dtypes, const sdr_dist* dists,
                       const sdr_rng* rngs, const sdr_view* views, int32_t n, void* stream);

/* Fused dropout on one window: keep-mask Bernoulli(1-p) (rng.py:238-242,
 * dispatch.py:567-576) applied as y = (x*m)*(1/(1-p)) (engine.py:80-81).
 * x, y: contiguous local tensors; y_dtype = x_dtype, or SDR_F32 for a BF16 x
 * (the reference's exact float32 result).  mask may be NULL; mask_dtype is
 * SDR_U8/SDR_BOOL or x_dtype.  Also serves the backward (gx = (gy*m)*s, the
 * mask regenerated from (seed, offset, view) instead of stored). */
int32_t sdr_dropout(const void* x, int32_t x_dtype, void* y, int32_t y_dtype, void* mask,
                    int32_t mask_dtype, double p, const sdr_rng* rng, const sdr_view* view,
                    void* stream);

/* NumPy transcendental mirror for Normal (rng.py:154-155): the float64 tables
 * L[k] = log1p(-k*2^-24) and c[k] = cos((2*pi)*(k*2^-24)) for k in [0, 2^24),
 * computed by the host's NumPy (host pointers; r = sqrt(-2 L) is correctly
 * rounded on both sides).  The tables are uploaded to `device` only while the
 * mirror is built: 2-bit ulp corrections of the device libm's log1p / cos
 * (8 MiB) plus a sorted exception list, verified bit for bit on all 2^24
 * points of both functions (if that ever fails, the full tables stay resident
 * instead).  Also calibrates the fast paths exhaustively and reports their max
 * errors (relative for r, absolute for c).  Reloading replaces the mirror. */
int32_t sdr_normal_tables_load(int32_t device, const double* log1p_table, const double* c_table,
                               double* max_rel_err_r, double* max_abs_err_c);
int32_t sdr_normal_tables_loaded(int32_t device);
/* Resident mirror bytes on `device`, exception count, 1 if the compact mirror
 * is in use (0: full tables), and the build time of the last load. */
int32_t sdr_normal_mirror_info(int32_t device, uint64_t* device_bytes, uint64_t* exceptions,
                               int32_t* compact, double* build_ms);
/* float64 Normal outputs read NumPy's r[k] as a fast function plus an 8-bit
 * correction per table point and c[k] from a double-double cosine that is
 * correctly rounded outside a flagged band (flagged points read an 8-bit
 * correction): 32 MiB, built and checked on all 2^24 points by
 * sdr_normal_tables_load (SDR_NORMAL_F64_DELTA=0 leaves them out and float64
 * normals take the mirror per element).  Reports their bytes on `device`
 * (0 when off), the points that escape to the mirror, and the largest stored
 * correction (in units of the last place) of each function.
 * No reference counterpart: rng.py:150-156 evaluates log1p / cos per element. */
int32_t sdr_normal_delta_info(int32_t device, uint64_t* device_bytes, uint64_t* escapes_r,
                              uint64_t* escapes_c, uint64_t* max_abs_r, uint64_t* max_abs_c);
/* Count of elements that took the exact (table) fallback since load. */
int32_t sdr_normal_fallback_count(int32_t device, uint64_t* count);

/* ---- pack / unpack for coalesced collectives (dtensor.py:261-298,
 *      comm.py:189-199, 269-279) ---------------------------------------- */

/* One member tensor of a coalesced collective.  The tensor is viewed as
 * [outer, rows, inner] (row-major, contiguous); along the middle dim it is
 * split into `nranks` chunks of `chunk_rows` rows (the last chunk may be
 * shorter / empty: ceil-block split, placement.py:226-231).  Rank-major packed
 * layout: packed[r][member m at byte offset seg_off[m]] holds chunk r of m,
 * padded to outer*chunk_rows*inner elements.  Members may mix dtypes for
 * gathers (bytes are moved); a reduce-scatter packs one dtype. */
typedef struct {
  void* data;           /* device pointer to the member tensor             */
  int64_t outer;        /* product of dims before the split dim            */
  int64_t rows;         /* extent of the split dim in `data`               */
  int64_t inner;        /* product of dims after the split dim             */
  int64_t chunk_rows;   /* ceil(global extent / nranks) along the split    */
  int64_t seg_off;      /* BYTE offset of this member inside one rank segment */
  int32_t elem_bytes;   /* 1, 2, 4 or 8                                     */
  int32_t pad_;
} sdr_pack_member;

/* Gather direction of a Shard->Replicate all-gather: scatter the packed
 * buffer (nranks segments of seg_elems elements) into full member tensors
 * (`rows` = full extent; member data = destination). */
int32_t sdr_unpack_gathered(const sdr_pack_member* members, int32_t n, const void* packed,
                            int64_t seg_bytes, int32_t nranks, void* stream);
/* Reduce-scatter input: copy full member tensors (Partial) into the
 * rank-major packed buffer so rank r's segment holds chunk r of every member. */
int32_t sdr_pack_scatter(const sdr_pack_member* members, int32_t n, void* packed,
                         int64_t seg_bytes, int32_t nranks, void* stream);
/* Copy this rank's shard of each member into (all_gather input) or out of
 * (reduce-scatter output) one contiguous segment. member.rows = local rows. */
int32_t sdr_pack_local(const sdr_pack_member* members, int32_t n, void* segment, void* stream);
int32_t sdr_unpack_local(const sdr_pack_member* members, int32_t n, const void* segment,
                         void* stream);
/* Replicate->Shard local slice (dtensor.py:247-251 via _local_slice,
 * dtensor.py:286-298): full[i] describes a tensor holding the whole split
 * extent (rows = extent, chunk_rows = ceil(extent/nranks)); piece[i].data
 * receives rank `rank`'s ceil-block rows (piece[i].rows = that row count,
 * same outer/inner/elem_bytes).  Also the slice step of Shard->Shard. */
int32_t sdr_slice_local(const sdr_pack_member* full, const sdr_pack_member* piece, int32_t n,
                        int32_t rank, int32_t nranks, void* stream);

/* ---- peer-memory collectives over NVLink / NVSwitch (CUDA IPC) ----------
 *
 * The fused redistribute without NCCL: every rank of a fiber owns a "peer
 * heap" (flag words + two data halves) that all fiber ranks map through CUDA
 * IPC.  A coalesced collective is then pack (local) -> sdr_peer_barrier ->
 * one pull kernel that reads every peer's half over NVLink and writes the
 * destination tensors directly:
 *   S->R  sdr_unpack_gathered_peers   (comm.py:104-110 + _assemble_shards,
 *                                      dtensor.py:261-283)
 *   P->S  sdr_reduce_scatter_peers    (comm.py:113-125 + _local_slice,
 *                                      dtensor.py:286-298)
 * The reduction sums in ascending fiber-rank order with one rounding per add,
 * in the tensor dtype, exactly like the reference's `acc += b` loop
 * (comm.py:120-122), including x86 NaN propagation: results are bit-exact for
 * any data, unlike a ring reduce-scatter.  Consecutive calls alternate the
 * two halves, so one barrier per call suffices (a rank reaches barrier k+1
 * only after its pull of call k).  Flags hold SDR_MAX_PEERS uint64 slots at
 * the heap base; slot q = the last epoch peer q arrived at. */
#define SDR_MAX_PEERS 64
#define SDR_PEER_FLAG_BYTES 4096

typedef struct { unsigned char bytes[64]; } sdr_ipc_handle;  /* cudaIpcMemHandle_t */

/* cudaMalloc `bytes` on `device` (flags zeroed) and export its IPC handle. */
int32_t sdr_peer_heap_alloc(int32_t device, int64_t bytes, void** base, sdr_ipc_handle* handle);
/* Map a peer's heap (another process) into this process on `device`. */
int32_t sdr_peer_heap_open(int32_t device, const sdr_ipc_handle* handle, void** base);
int32_t sdr_peer_heap_close(void* base);  /* unmap a peer heap */
int32_t sdr_peer_heap_free(void* base);   /* free this process's own heap */
/* Device-side barrier of `nranks` fiber ranks: stores `epoch` (release, system
 * scope) into slot `rank` of every rank's flags, then waits (acquire) until
 * every slot of flags[rank] >= epoch.  epoch == 0 takes the epoch from the
 * device: this rank's barrier counter (flag word SDR_MAX_PEERS + 1 of its own
 * heap) + 1, stored back -- the form a captured CUDA graph can replay; a heap
 * must use one form or the other, not both.  flags: host array of nranks device
 * pointers (each rank's heap base).  A wait longer than timeout_ns traps (the
 * call fails loudly instead of hanging).  timeout_ns < 0 is the soft mode of
 * the transport's self-check: after |timeout_ns| the kernel sets flag word
 * SDR_MAX_PEERS of this rank's own heap to 1 and returns (no trap). */
int32_t sdr_peer_barrier(void* const* flags, int32_t rank, int32_t nranks, uint64_t epoch,
                         int64_t timeout_ns, void* stream);
/* Synchronous read of flag word `index` of a heap (e.g. the soft-timeout word
 * SDR_MAX_PEERS after a self-check). */
int32_t sdr_peer_flag_read(const void* base, int32_t index, uint64_t* value);
/* S->R pull: segment r of the gathered layout (sdr_unpack_gathered) is read
 * from segs[r] (rank r's packed shard, usually in its peer heap). */
int32_t sdr_unpack_gathered_peers(const sdr_pack_member* members, int32_t n,
                                  const void* const* segs, int32_t nranks, void* stream);
/* P->S pull: members are this rank's OUTPUT pieces (rows = this rank's rows,
 * as sdr_unpack_local); packed[q] is rank q's rank-major packed buffer
 * (sdr_pack_scatter).  out = sum over q ascending of packed[q] segment `rank`,
 * in `dtype` (SDR_F32/F64/BF16/F16/I32/I64). */
int32_t sdr_reduce_scatter_peers(const sdr_pack_member* members, int32_t n,
                                 const void* const* packed, int64_t seg_bytes, int32_t nranks,
                                 int32_t rank, int32_t dtype, void* stream);

/* One whole peer collective per call (what the redistribute plan replays):
 * the three launches above behind one entry point, with the segments at
 * bases[q] + half_offset.  lead_barrier != 0 adds a barrier BEFORE the pack
 * (same epoch rule, epoch + 0 / device epoch): every peer has then finished
 * its pulls of earlier calls from this half, whatever half they used -- the
 * mode for calls inside (or interleaved with) captured CUDA graphs, whose
 * replays the host does not see.  With epoch != 0 the lead barrier uses
 * epoch and the main one epoch + 1.  S->R: sdr_pack_local(send -> my segment),
 * sdr_peer_barrier(epoch), sdr_unpack_gathered_peers(recv). */
int32_t sdr_peer_all_gather(const sdr_pack_member* send, const sdr_pack_member* recv, int32_t n,
                            void* const* bases, int32_t nranks, int32_t rank, int64_t half_offset,
                            uint64_t epoch, int64_t timeout_ns, int32_t lead_barrier, void* stream);
/* P->S: sdr_pack_scatter(full -> my half, seg_bytes per rank),
 * sdr_peer_barrier(epoch), sdr_reduce_scatter_peers(piece). */
int32_t sdr_peer_reduce_scatter(const sdr_pack_member* full, const sdr_pack_member* piece, int32_t n,
                                void* const* bases, int32_t nranks, int32_t rank, int64_t half_offset,
                                int64_t seg_bytes, int32_t dtype, uint64_t epoch, int64_t timeout_ns,
                                int32_t lead_barrier, void* stream);

/* INT32 pipe microbenchmark: measured IMAD.WIDE.U32 and LOP3 throughput
 * (ops/s) on `device`, for the roofline denominator. */
int32_t sdr_probe_int32(int32_t device, double* imad_wide_per_s, double* lop3_per_s,
                        double* philox_blocks_per_s);

#ifdef __cplusplus
}
#endif

#endif /* SDRNG_H_ */
