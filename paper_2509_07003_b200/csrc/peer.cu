// peer.cu -- fused redistribute collectives over NVLink / NVSwitch peer memory.
//
// The NCCL path of a coalesced collective is pack -> NCCL -> unpack (three
// passes, two of them local copies).  Here the fiber ranks map each other's
// "peer heap" (CUDA IPC) and a collective is:
//   pack into my heap half (k_copy_tiles) -> k_peer_barrier -> ONE pull kernel
// whose CTAs read the peers' halves over NVLink and write the destination
// tensors directly.  S->R pulls with the copy kernel itself (source pointers
// per rank segment); P->S pulls with k_reduce_peers, which sums the P
// segments in ascending fiber-rank order, one rounding per add, in the tensor
// dtype -- the reference's `acc = b0.copy(); acc += b1; ...` (comm.py:120-122)
// bit for bit, x86 NaN propagation included.
#include <cstdio>
#include <utility>

#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "copy_tiles.cuh"

namespace sdr {

// ---- NumPy-exact elementwise a + b (x86 SSE/AVX NaN rules: a NaN operand
// propagates quieted, first operand first; an invalid op gives the negative
// default NaN) ----------------------------------------------------------------
__device__ __forceinline__ uint32_t add_f32(uint32_t a, uint32_t b) {
  const float fa = __uint_as_float(a), fb = __uint_as_float(b);
  const float r = __fadd_rn(fa, fb);
  if (r != r) {
    if (fa != fa) return a | 0x00400000u;
    if (fb != fb) return b | 0x00400000u;
    return 0xFFC00000u;
  }
  return __float_as_uint(r);
}

__device__ __forceinline__ uint64_t add_f64(uint64_t a, uint64_t b) {
  const double fa = __longlong_as_double(static_cast<long long>(a));
  const double fb = __longlong_as_double(static_cast<long long>(b));
  const double r = __dadd_rn(fa, fb);
  if (r != r) {
    if (fa != fa) return a | 0x0008000000000000ull;
    if (fb != fb) return b | 0x0008000000000000ull;
    return 0xFFF8000000000000ull;
  }
  return static_cast<uint64_t>(__double_as_longlong(r));
}

// bfloat16 (ml_dtypes): float32 add, then RNE to bfloat16; NaN -> sign|0x7FC0.
__device__ __forceinline__ uint16_t add_bf16(uint16_t a, uint16_t b) {
  const float fa = __uint_as_float(static_cast<uint32_t>(a) << 16);
  const float fb = __uint_as_float(static_cast<uint32_t>(b) << 16);
  const float r = __fadd_rn(fa, fb);
  if (r != r) {
    const uint16_t s = fa != fa ? (a & 0x8000u) : fb != fb ? (b & 0x8000u) : 0x8000u;
    return static_cast<uint16_t>(s | 0x7FC0u);
  }
  uint32_t u = __float_as_uint(r);
  u += 0x7FFFu + ((u >> 16) & 1u);
  return static_cast<uint16_t>(u >> 16);
}

// float16 (NumPy npy_half): float32 add, then RNE to half; a NaN keeps its
// top mantissa bits with the quiet bit set.
__device__ __forceinline__ uint16_t add_f16(uint16_t a, uint16_t b) {
  const float fa = __half2float(__ushort_as_half(a));
  const float fb = __half2float(__ushort_as_half(b));
  const float r = __fadd_rn(fa, fb);
  if (r != r) {
    if (fa != fa) return static_cast<uint16_t>(a | 0x0200u);
    if (fb != fb) return static_cast<uint16_t>(b | 0x0200u);
    return 0xFE00u;
  }
  return __half_as_ushort(__float2half_rn(r));
}

template <int DT> struct Elem;
template <> struct Elem<SDR_F32> {
  using T = uint32_t;
  static __device__ __forceinline__ T add(T a, T b) { return add_f32(a, b); }
};
template <> struct Elem<SDR_F64> {
  using T = uint64_t;
  static __device__ __forceinline__ T add(T a, T b) { return add_f64(a, b); }
};
template <> struct Elem<SDR_BF16> {
  using T = uint16_t;
  static __device__ __forceinline__ T add(T a, T b) { return add_bf16(a, b); }
};
template <> struct Elem<SDR_F16> {
  using T = uint16_t;
  static __device__ __forceinline__ T add(T a, T b) { return add_f16(a, b); }
};
template <> struct Elem<SDR_I32> {
  using T = uint32_t;  // two's-complement wrap, as NumPy int32
  static __device__ __forceinline__ T add(T a, T b) { return a + b; }
};
template <> struct Elem<SDR_I64> {
  using T = uint64_t;
  static __device__ __forceinline__ T add(T a, T b) { return a + b; }
};

template <int DT, typename V>
__device__ __forceinline__ void vadd(V& acc, const V& x) {
  using T = typename Elem<DT>::T;
  constexpr int k = sizeof(V) / sizeof(T);
  T a[k], b[k];
  memcpy(a, &acc, sizeof(V));
  memcpy(b, &x, sizeof(V));
#pragma unroll
  for (int i = 0; i < k; ++i) a[i] = Elem<DT>::add(a[i], b[i]);
  memcpy(&acc, a, sizeof(V));
}

// Programmatic dependent launch along pack -> barrier -> pull: the barrier and
// the pull are launched with programmatic stream serialization, so their
// launch overlaps the previous kernel; each executes griddepcontrol.wait (all
// prerequisite grids complete, memory visible) before touching memory.
#ifndef SDR_PEER_PDL
#define SDR_PEER_PDL 1
#endif

__device__ __forceinline__ void pdl_wait() {
#if SDR_PEER_PDL
  asm volatile("griddepcontrol.wait;" ::: "memory");
#endif
}

template <typename... KArgs, typename... Args>
static void launch_dep(void (*kernel)(KArgs...), unsigned grid, unsigned block, cudaStream_t s,
                       Args&&... args) {
#if SDR_PEER_PDL
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
#else
  kernel<<<grid, block, 0, s>>>(std::forward<Args>(args)...);
#endif
}

#ifndef SDR_REDUCE_MINB
#define SDR_REDUCE_MINB 5  // 48 regs: 5 CTAs per SM (latency-bound pull; A/B: 1 -> 4.4, 5 -> 5.1 TB/s at P=2)
#endif

#ifndef SDR_REDUCE_TILE
#define SDR_REDUCE_TILE 16384
#endif
#ifndef SDR_REDUCE_PAIRS
#define SDR_REDUCE_PAIRS 0  // two peers per load round (A/B: no gain, profiles/r01_peer_reduce_tile_ab.txt)
#endif
constexpr int64_t kReduceTile = SDR_REDUCE_TILE;

// Loads of peer memory bypass the caches (ld.global.cv): a half is rewritten
// by its owner every other call, so no line of it may be reused from a cache
// across calls; the owner's L2 is the point of coherence.
template <typename V>
__device__ __forceinline__ V load_peer(const unsigned char* p) {
  return __ldcv(reinterpret_cast<const V*>(p));
}

struct PeerPtrs {
  const unsigned char* p[SDR_MAX_PEERS];
};

// One CTA per <= kReduceTile tile of the output pieces.  Job `src` fields are
// byte OFFSETS into every rank's packed buffer (same layout on every rank).
// All U loads of one peer are issued before they are summed, so each thread
// keeps U NVLink reads in flight.
template <int DT, typename V>
__global__ void __launch_bounds__(256, SDR_REDUCE_MINB) k_reduce_peers(const __grid_constant__ JobTable T,
                                                      const __grid_constant__ PeerPtrs B,
                                                      int nranks) {
  constexpr int U = static_cast<int>(kReduceTile / (sizeof(V) * 256));
  const unsigned char* so[U];
  unsigned char* dv[U];
  const int total = tile_slots<V, U>(T.jobs, T.prefix, T.n, so, dv);
  pdl_wait();
  V acc[U];
#pragma unroll
  for (int u = 0; u < U; ++u)
    if (static_cast<int>(threadIdx.x) + u * 256 < total)
      acc[u] = load_peer<V>(B.p[0] + reinterpret_cast<uintptr_t>(so[u]));
  int q = 1;
#if SDR_REDUCE_PAIRS
  for (; q + 1 < nranks; q += 2) {  // two peers per round: 2U loads in flight
    V x[U], y[U];
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (static_cast<int>(threadIdx.x) + u * 256 < total) {
        x[u] = load_peer<V>(B.p[q] + reinterpret_cast<uintptr_t>(so[u]));
        y[u] = load_peer<V>(B.p[q + 1] + reinterpret_cast<uintptr_t>(so[u]));
      }
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (static_cast<int>(threadIdx.x) + u * 256 < total) {
        vadd<DT>(acc[u], x[u]);
        vadd<DT>(acc[u], y[u]);
      }
  }
#endif
  for (; q < nranks; ++q) {
    V x[U];
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (static_cast<int>(threadIdx.x) + u * 256 < total)
        x[u] = load_peer<V>(B.p[q] + reinterpret_cast<uintptr_t>(so[u]));
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (static_cast<int>(threadIdx.x) + u * 256 < total) vadd<DT>(acc[u], x[u]);
  }
#pragma unroll
  for (int u = 0; u < U; ++u)
    if (static_cast<int>(threadIdx.x) + u * 256 < total) *reinterpret_cast<V*>(dv[u]) = acc[u];
}

// Gather pull: the plain copy over per-segment peer source pointers.
template <typename V>
__global__ void __launch_bounds__(256) k_gather_peers(const __grid_constant__ JobTable T) {
  constexpr int U = static_cast<int>(kTileBytes / (sizeof(V) * 256));
  const unsigned char* sv[U];
  unsigned char* dv[U];
  const int total = tile_slots<V, U>(T.jobs, T.prefix, T.n, sv, dv);
  pdl_wait();
  V v[U];
#pragma unroll
  for (int u = 0; u < U; ++u)
    if (static_cast<int>(threadIdx.x) + u * 256 < total) v[u] = load_peer<V>(sv[u]);
#pragma unroll
  for (int u = 0; u < U; ++u)
    if (static_cast<int>(threadIdx.x) + u * 256 < total) *reinterpret_cast<V*>(dv[u]) = v[u];
}

struct PeerFlags {
  unsigned long long* p[SDR_MAX_PEERS];
};

// Thread t: announce arrival in rank t's slot `rank`, then wait for rank t's
// arrival in my slot t.  The fence orders every write of the preceding
// kernels on this stream (the pack) before the release store.
__global__ void k_peer_barrier(const __grid_constant__ PeerFlags F, int rank, int nranks,
                               unsigned long long epoch, long long timeout_ns) {
  pdl_wait();  // the pack before us has completed and is visible
  // No early trigger: the pull's CTAs would sit resident in griddepcontrol.wait
  // on every SM while we spin, starving other streams of the same GPU (with
  // ranks as streams of one GPU that deadlocks: tests/test_peer_gpu.py).
  const int t = threadIdx.x;
  if (epoch == 0) {
    // device epoch: this rank's barrier counter (flag word SDR_MAX_PEERS + 1
    // of its own heap, touched by no other rank) advances once per barrier,
    // so a CUDA graph that captured this launch replays with fresh epochs;
    // every fiber rank runs the same barrier sequence, so the counters agree
    __shared__ unsigned long long s_epoch;
    if (t == 0) s_epoch = atomicAdd(F.p[rank] + SDR_MAX_PEERS + 1, 1ull) + 1ull;
    __syncthreads();
    epoch = s_epoch;
  }
  if (t >= nranks) return;
  asm volatile("fence.acq_rel.sys;" ::: "memory");
  // max, not a plain store: a slot's epoch can never move backwards, whatever
  // order two barrier kernels of this rank happen to run in
  asm volatile("red.release.sys.global.max.u64 [%0], %1;" ::"l"(F.p[t] + rank), "l"(epoch) : "memory");
  const unsigned long long* mine = F.p[rank] + t;
  unsigned long long t0, now, v;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (;;) {
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(mine) : "memory");
    if (v >= epoch) break;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
    if (static_cast<long long>(now - t0) > (timeout_ns < 0 ? -timeout_ns : timeout_ns)) {
      if (timeout_ns < 0) {  // soft mode: record the timeout in my own flag word SDR_MAX_PEERS, return
        atomicMax(F.p[rank] + SDR_MAX_PEERS, 1ull);
        return;
      }
      printf("sdr_peer_barrier: rank %d timed out waiting for fiber rank %d (epoch %llu, saw %llu)\n",
             rank, t, epoch, v);
      __trap();
    }
    __nanosleep(100);
  }
}

// Launch a job list in groups of <= kParamJobs (job table as a kernel
// parameter: no allocation per call, graph-capturable).
template <class Launch>
static int launch_groups(const std::vector<CopyJob>& jobs, Launch&& launch) {
  for (size_t g = 0; g < jobs.size(); g += kParamJobs) {
    const int n = static_cast<int>(std::min(jobs.size() - g, static_cast<size_t>(kParamJobs)));
    JobTable T;
    memset(static_cast<void*>(&T), 0, sizeof(T));
    T.n = n;
    int64_t tiles = 0;
    int vec = 16;
    for (int i = 0; i < n; ++i) {
      T.prefix[i] = tiles;
      T.jobs[i] = jobs[g + i];
      tiles += T.jobs[i].tiles;
      vec = T.jobs[i].vec < vec ? T.jobs[i].vec : vec;
    }
    if (tiles == 0) continue;
    launch(T, static_cast<unsigned>(tiles), vec);
    const int st = check_launch();
    if (st != SDR_OK) return st;
  }
  return SDR_OK;
}

int unpack_gathered_peers(const sdr_pack_member* M, int n, const void* const* segs, int nranks,
                          cudaStream_t s) {
  if (n < 0 || nranks < 1 || nranks > SDR_MAX_PEERS || (n > 0 && (M == nullptr || segs == nullptr)))
    return SDR_E_INVALID;
  for (int r = 0; r < nranks && n > 0; ++r)
    if (segs[r] == nullptr) return SDR_E_INVALID;
  std::vector<CopyJob> jobs;
  for (int i = 0; i < n; ++i) {
    const sdr_pack_member& m = M[i];
    if (!member_ok(m) || m.chunk_rows * nranks < m.rows) return SDR_E_INVALID;
    const int64_t row_b = m.inner * m.elem_bytes;
    for (int r = 0; r < nranks; ++r) {
      int64_t lo, len;
      rank_rows(m.rows, m.chunk_rows, r, lo, len);
      add_job(jobs, static_cast<const unsigned char*>(segs[r]) + m.seg_off,
              static_cast<unsigned char*>(m.data) + lo * row_b, m.outer, len * row_b,
              m.chunk_rows * row_b, m.rows * row_b);
    }
  }
  return launch_groups(jobs, [&](const JobTable& T, unsigned grid, int vec) {
    switch (vec) {
      case 16: launch_dep(k_gather_peers<uint4>, grid, 256, s, T); break;
      case 8: launch_dep(k_gather_peers<uint2>, grid, 256, s, T); break;
      case 4: launch_dep(k_gather_peers<uint32_t>, grid, 256, s, T); break;
      case 2: launch_dep(k_gather_peers<uint16_t>, grid, 256, s, T); break;
      default: launch_dep(k_gather_peers<unsigned char>, grid, 256, s, T); break;
    }
  });
}

template <int DT>
static void launch_reduce(const JobTable& T, unsigned grid, int vec, const PeerPtrs& B,
                          int nranks, cudaStream_t s) {
  using E = typename Elem<DT>::T;
  if (vec >= 16) {
    launch_dep(k_reduce_peers<DT, uint4>, grid, 256, s, T, B, nranks);
  } else if (vec >= 8) {
    launch_dep(k_reduce_peers<DT, uint2>, grid, 256, s, T, B, nranks);
  } else if constexpr (sizeof(E) <= 4) {
    if (vec >= 4) launch_dep(k_reduce_peers<DT, uint32_t>, grid, 256, s, T, B, nranks);
    else if constexpr (sizeof(E) <= 2) launch_dep(k_reduce_peers<DT, uint16_t>, grid, 256, s, T, B, nranks);
  }
}

int reduce_scatter_peers(const sdr_pack_member* M, int n, const void* const* packed,
                         int64_t seg_bytes, int nranks, int rank, int dtype, cudaStream_t s) {
  if (n < 0 || nranks < 1 || nranks > SDR_MAX_PEERS || rank < 0 || rank >= nranks ||
      seg_bytes < 0 || (n > 0 && (M == nullptr || packed == nullptr)))
    return SDR_E_INVALID;
  int es;
  switch (dtype) {
    case SDR_F32: case SDR_I32: es = 4; break;
    case SDR_F64: case SDR_I64: es = 8; break;
    case SDR_BF16: case SDR_F16: es = 2; break;
    default: return SDR_E_DTYPE;
  }
  PeerPtrs B;
  memset(&B, 0, sizeof(B));
  for (int q = 0; q < nranks; ++q) {
    if (n > 0 && packed[q] == nullptr) return SDR_E_INVALID;
    if (reinterpret_cast<uintptr_t>(packed[q]) % 16 != 0) return SDR_E_ALIGN;
    B.p[q] = static_cast<const unsigned char*>(packed[q]);
  }
  std::vector<CopyJob> jobs;
  for (int i = 0; i < n; ++i) {
    const sdr_pack_member& m = M[i];
    if (!member_ok(m) || m.elem_bytes != es || m.rows > m.chunk_rows) return SDR_E_INVALID;
    const int64_t row_b = m.inner * es;
    if (m.seg_off + m.outer * m.chunk_rows * row_b > seg_bytes) return SDR_E_INVALID;
    // source = offset of my segment's slot inside every rank's packed buffer
    const uintptr_t off = static_cast<uintptr_t>(rank * seg_bytes + m.seg_off);
    add_job(jobs, reinterpret_cast<const void*>(off), m.data, m.outer, m.rows * row_b,
            m.chunk_rows * row_b, m.rows * row_b, kReduceTile);
  }
  for (const CopyJob& J : jobs)
    if (J.vec < es) return SDR_E_ALIGN;
  return launch_groups(jobs, [&](const JobTable& T, unsigned grid, int vec) {
    switch (dtype) {
      case SDR_F32: launch_reduce<SDR_F32>(T, grid, vec, B, nranks, s); break;
      case SDR_F64: launch_reduce<SDR_F64>(T, grid, vec, B, nranks, s); break;
      case SDR_BF16: launch_reduce<SDR_BF16>(T, grid, vec, B, nranks, s); break;
      case SDR_F16: launch_reduce<SDR_F16>(T, grid, vec, B, nranks, s); break;
      case SDR_I32: launch_reduce<SDR_I32>(T, grid, vec, B, nranks, s); break;
      default: launch_reduce<SDR_I64>(T, grid, vec, B, nranks, s); break;
    }
  });
}

int peer_barrier(void* const* flags, int rank, int nranks, uint64_t epoch, int64_t timeout_ns,
                 cudaStream_t s) {
  if (flags == nullptr || nranks < 1 || nranks > SDR_MAX_PEERS || rank < 0 || rank >= nranks ||
      timeout_ns == 0)
    return SDR_E_INVALID;
  PeerFlags F;
  memset(&F, 0, sizeof(F));
  for (int q = 0; q < nranks; ++q) {
    if (flags[q] == nullptr) return SDR_E_INVALID;
    F.p[q] = static_cast<unsigned long long*>(flags[q]);
  }
  launch_dep(k_peer_barrier, 1u, 32u * ((nranks + 31) / 32), s, F, rank, nranks,
             static_cast<unsigned long long>(epoch), static_cast<long long>(timeout_ns));
  return check_launch();
}

// ---- heap management (host) ----------------------------------------------
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

static int cuda_status(cudaError_t e) {
  if (e == cudaSuccess) return SDR_OK;
  set_cuda_error(e);
  return SDR_E_CUDA;
}

int peer_flag_read(const void* base, int index, uint64_t* value) {
  if (base == nullptr || value == nullptr || index < 0 || index >= SDR_PEER_FLAG_BYTES / 8)
    return SDR_E_INVALID;
  return cuda_status(cudaMemcpy(value, static_cast<const uint64_t*>(base) + index, 8, cudaMemcpyDeviceToHost));
}


int preload_copy_kernels();

// Load every kernel a peer collective launches (see preload_copy_kernels):
// behind a spinning barrier, a lazy load at the pull's first launch would
// stall this rank's host thread -- and deadlock ranks driven by one thread.
static int preload_peer_kernels() {
  int st = preload_copy_kernels();
  if (st != SDR_OK) return st;
  cudaFuncAttributes a;
  const void* fns[] = {
      reinterpret_cast<const void*>(&k_peer_barrier),
      reinterpret_cast<const void*>(&k_gather_peers<uint4>), reinterpret_cast<const void*>(&k_gather_peers<uint2>),
      reinterpret_cast<const void*>(&k_gather_peers<uint32_t>), reinterpret_cast<const void*>(&k_gather_peers<uint16_t>),
      reinterpret_cast<const void*>(&k_gather_peers<unsigned char>),
#define SDR_RP(DT) reinterpret_cast<const void*>(&k_reduce_peers<DT, uint4>), \
      reinterpret_cast<const void*>(&k_reduce_peers<DT, uint2>)
      SDR_RP(SDR_F32), SDR_RP(SDR_F64), SDR_RP(SDR_BF16), SDR_RP(SDR_F16), SDR_RP(SDR_I32), SDR_RP(SDR_I64),
#undef SDR_RP
      reinterpret_cast<const void*>(&k_reduce_peers<SDR_F32, uint32_t>),
      reinterpret_cast<const void*>(&k_reduce_peers<SDR_I32, uint32_t>),
      reinterpret_cast<const void*>(&k_reduce_peers<SDR_BF16, uint32_t>),
      reinterpret_cast<const void*>(&k_reduce_peers<SDR_F16, uint32_t>),
      reinterpret_cast<const void*>(&k_reduce_peers<SDR_BF16, uint16_t>),
      reinterpret_cast<const void*>(&k_reduce_peers<SDR_F16, uint16_t>)};
  for (const void* f : fns) {
    const cudaError_t e = cudaFuncGetAttributes(&a, f);
    if (e != cudaSuccess) return cuda_status(e);
  }
  return SDR_OK;
}

int peer_heap_alloc(int device, int64_t bytes, void** base, sdr_ipc_handle* handle) {
  static_assert(sizeof(sdr_ipc_handle) == sizeof(cudaIpcMemHandle_t), "IPC handle size");
  if (base == nullptr || handle == nullptr || bytes < SDR_PEER_FLAG_BYTES) return SDR_E_INVALID;
  DeviceGuard g(device);
  const int pst = preload_peer_kernels();
  if (pst != SDR_OK) return pst;
  void* p = nullptr;
  int st = cuda_status(cudaMalloc(&p, static_cast<size_t>(bytes)));
  if (st != SDR_OK) return st;
  st = cuda_status(cudaMemset(p, 0, SDR_PEER_FLAG_BYTES));
  cudaIpcMemHandle_t h;
  if (st == SDR_OK) st = cuda_status(cudaIpcGetMemHandle(&h, p));
  if (st == SDR_OK) st = cuda_status(cudaDeviceSynchronize());
  if (st != SDR_OK) {
    cudaFree(p);
    return st;
  }
  memcpy(handle->bytes, &h, sizeof(h));
  *base = p;
  return SDR_OK;
}

int peer_heap_open(int device, const sdr_ipc_handle* handle, void** base) {
  if (base == nullptr || handle == nullptr) return SDR_E_INVALID;
  DeviceGuard g(device);
  cudaIpcMemHandle_t h;
  memcpy(&h, handle->bytes, sizeof(h));
  return cuda_status(cudaIpcOpenMemHandle(base, h, cudaIpcMemLazyEnablePeerAccess));
}

int peer_heap_close(void* base) { return cuda_status(cudaIpcCloseMemHandle(base)); }

int peer_heap_free(void* base) { return cuda_status(cudaFree(base)); }

}  // namespace sdr
