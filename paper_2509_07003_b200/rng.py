"""Single-device-semantic distributed RNG on B200 (sm_100a).

Drop-in API mirror of spmdsim.rng (reference: /root/reference/pkg/src/spmdsim/
rng.py:1-265).  Every value is a pure function of (seed, offset, THETA, j), j
the element's global row-major flat index: tau = j mod THETA,
beta = j div THETA + offset, one Philox4x32-10 block per element on counter
(beta_lo, beta_hi, tau_lo, tau_hi) with key (seed_lo, seed_hi).  So each rank
generates exactly its window of the unsharded tensor, with no communication.

All arithmetic runs in the sm_100a kernels of `libsdrng.so` (via `_lib`);
results are torch tensors on the CUDA device.  The shared state is three
integers advanced on the host exactly like rng.py:95-98, once per op, on every
rank, with no collective.

Differences in representation (not in values):
  * outputs are torch tensors; NumPy / ml_dtypes dtypes are accepted and mapped
    (np.float32 -> torch.float32, ml_dtypes.bfloat16 -> torch.bfloat16, ...);
  * user-defined Distribution subclasses cannot run (no CPU fallback): only
    the five reference distributions have kernels.
"""

from __future__ import annotations

import ctypes as C
import math
import threading
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .placement import ShardSpec, ShardView, full_view, local_shape_and_offset

DEFAULT_GLOBAL_THREADS = 65536


# ---------------------------------------------------------------------------
# Generator state (reference rng.py:85-101)
# ---------------------------------------------------------------------------
@dataclass
class RngState:
    seed: int = 0
    offset: int = 0
    global_threads: int = DEFAULT_GLOBAL_THREADS

    def __post_init__(self):
        if self.global_threads < 1:
            raise ValueError("global thread count must be >= 1")

    def advance(self, global_numel: int, blocks_per_element: int = 1):
        """offset += ceil(global_numel / THETA) * K -- identical on every rank,
        for empty local shards too."""
        self.offset += -(-int(global_numel) // self.global_threads) * blocks_per_element

    def clone(self) -> "RngState":
        return RngState(self.seed, self.offset, self.global_threads)

    def native(self) -> _lib.SdrRng:
        r = _lib.SdrRng()
        r.seed = int(self.seed) & 0xFFFFFFFFFFFFFFFF
        r.offset = int(self.offset) & 0xFFFFFFFFFFFFFFFF
        r.theta = int(self.global_threads)
        return r


# ---------------------------------------------------------------------------
# dtypes
# ---------------------------------------------------------------------------
_TORCH_OF_CODE = {
    _lib.F32: torch.float32, _lib.F64: torch.float64, _lib.BF16: torch.bfloat16,
    _lib.F16: torch.float16, _lib.I64: torch.int64, _lib.I32: torch.int32,
    _lib.U8: torch.uint8, _lib.BOOL: torch.bool,
}
_CODE_OF_TORCH = {v: k for k, v in _TORCH_OF_CODE.items()}
_CODE_OF_NAME = {
    "float32": _lib.F32, "float64": _lib.F64, "bfloat16": _lib.BF16, "float16": _lib.F16,
    "int64": _lib.I64, "int32": _lib.I32, "uint8": _lib.U8, "bool": _lib.BOOL,
}


def dtype_code(dtype) -> int:
    """sdr_dtype code for a torch / NumPy / ml_dtypes dtype (or its name)."""
    if dtype is None:
        return _lib.F64
    if isinstance(dtype, torch.dtype):
        if dtype not in _CODE_OF_TORCH:
            raise TypeError(f"unsupported dtype {dtype}")
        return _CODE_OF_TORCH[dtype]
    name = dtype if isinstance(dtype, str) else np.dtype(dtype).name
    if name not in _CODE_OF_NAME:
        raise TypeError(f"unsupported dtype {dtype!r}")
    return _CODE_OF_NAME[name]


def torch_dtype(dtype) -> torch.dtype:
    return _TORCH_OF_CODE[dtype_code(dtype)]


# ---------------------------------------------------------------------------
# Distributions (reference rng.py:104-182).  `transform` runs on the GPU.
# ---------------------------------------------------------------------------
class Distribution:
    """Maps one Philox block to one value; no cross-element state."""

    blocks_per_element = 1
    kind: int | None = None

    def native(self) -> _lib.SdrDist:
        raise TypeError(f"{type(self).__name__} has no sm_100a kernel (no CPU fallback)")

    def out_code(self, code: int) -> int:
        """Output dtype code the reference produces for requested `code`."""
        return code

    def transform(self, words, dtype=np.float64):
        """Values for Philox words (4 uint32 arrays/tensors), computed on GPU."""
        return transform_words(self, words, dtype)


class Uniform01(Distribution):
    """float32: (w0 >> 8) * 2^-24.  Any other dtype: 53 bits of words 0-1 as
    float64 -- the reference returns float64 there (rng.py:124-127)."""

    kind = _lib.UNIFORM01

    def native(self):
        d = _lib.SdrDist()
        d.kind = self.kind
        return d

    def out_code(self, code):
        return _lib.F32 if code == _lib.F32 else _lib.F64


class Uniform(Distribution):
    """lo + (hi - lo) * u: float32 arithmetic on the 24-bit u for float32,
    float64 on the 53-bit u then one cast otherwise (rng.py:130-138)."""

    kind = _lib.UNIFORM

    def __init__(self, lo: float = 0.0, hi: float = 1.0):
        if not lo < hi:
            raise ValueError(f"uniform needs lo < hi, got [{lo}, {hi})")
        self.lo, self.hi = lo, hi

    def native(self):
        # The library forms hi - lo in float64, which equals the reference's
        # Python arithmetic for floats and for integers up to 2**53.
        for v in (self.lo, self.hi, self.hi - self.lo):
            if isinstance(v, int) and abs(v) > 2 ** 53:
                raise TypeError("Uniform bounds beyond 2**53 are not supported on GPU")
        d = _lib.SdrDist()
        d.kind = self.kind
        d.fparam[0] = float(self.lo)
        d.fparam[1] = float(self.hi)
        return d


class Normal(Distribution):
    """Box-Muller on words 0 and 1 (rng.py:141-156), float64, then one cast."""

    kind = _lib.NORMAL

    def __init__(self, mean: float = 0.0, std: float = 1.0):
        if std <= 0:
            raise ValueError("std must be positive")
        self.mean, self.std = mean, std

    def native(self):
        d = _lib.SdrDist()
        d.kind = self.kind
        d.fparam[0] = float(self.mean)
        d.fparam[1] = float(self.std)
        return d


class RandInt(Distribution):
    """lo + (64-bit draw from words 0-1) mod (hi - lo) (rng.py:159-171)."""

    kind = _lib.RANDINT

    def __init__(self, lo: int, hi: int):
        if not lo < hi:
            raise ValueError(f"randint needs lo < hi, got [{lo}, {hi})")
        self.lo, self.hi = lo, hi

    def native(self):
        d = _lib.SdrDist()
        d.kind = self.kind
        d.iparam[0] = int(self.lo)
        d.iparam[1] = int(self.hi)
        return d


class Bernoulli(Distribution):
    """1 where the 53-bit uniform of words 0-1 is < p (rng.py:174-182)."""

    kind = _lib.BERNOULLI

    def __init__(self, p: float):
        if not 0.0 <= p <= 1.0:
            raise ValueError(f"p must be in [0, 1], got {p}")
        self.p = p

    def native(self):
        d = _lib.SdrDist()
        d.kind = self.kind
        d.fparam[0] = float(self.p)
        return d


# ---------------------------------------------------------------------------
# NumPy transcendental mirror for Normal
# ---------------------------------------------------------------------------
_TABLES_LOCK = threading.Lock()
_TABLE_ERRORS: dict[int, tuple[float, float]] = {}


def numpy_normal_tables() -> tuple[np.ndarray, np.ndarray]:
    """L[k] = log1p(-u), c[k] = cos(2*pi*u), u = k*2^-24, k < 2^24, evaluated
    with the same NumPy expressions as rng.py:152-155 on this host (the
    reference's r is sqrt(-2.0 * L), correctly rounded, so L pins it)."""
    u = np.arange(1 << 24, dtype=np.uint32).astype(np.float64) * 2.0 ** -24
    L = np.log1p(-u)
    c = np.cos(2.0 * np.pi * u)
    return np.ascontiguousarray(L), np.ascontiguousarray(c)


def ensure_normal_tables(device=None) -> tuple[float, float]:
    """Load (once per device) the NumPy mirror tables used to certify/round
    the float64 Box-Muller exactly as the reference's NumPy does."""
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    idx = dev.index if dev.index is not None else torch.cuda.current_device()
    with _TABLES_LOCK:
        if idx in _TABLE_ERRORS and _lib.LIB.sdr_normal_tables_loaded(idx):
            return _TABLE_ERRORS[idx]
        L, c = numpy_normal_tables()
        er, ec = C.c_double(), C.c_double()
        st = _lib.LIB.sdr_normal_tables_load(idx, L.ctypes.data, c.ctypes.data, C.byref(er), C.byref(ec))
        _lib.check(st, "sdr_normal_tables_load")
        _TABLE_ERRORS[idx] = (er.value, ec.value)
        return _TABLE_ERRORS[idx]


def normal_mirror_info(device=None) -> dict:
    """Resident bytes of the Normal mirror on `device`, its exception count,
    whether the compact (2-bit correction) form is in use, and the build time
    of the device part of the last load (ms)."""
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    idx = dev.index if dev.index is not None else torch.cuda.current_device()
    nb, nx, cp, ms = C.c_uint64(), C.c_uint64(), C.c_int32(), C.c_double()
    _lib.check(_lib.LIB.sdr_normal_mirror_info(idx, C.byref(nb), C.byref(nx), C.byref(cp), C.byref(ms)),
               "sdr_normal_mirror_info")
    return {"device_bytes": nb.value, "exceptions": nx.value, "compact": bool(cp.value),
            "build_ms": ms.value}


def normal_delta_info(device=None) -> dict:
    """The float64 Normal corrections on `device` (sdr_normal_delta_info):
    resident bytes (0 when SDR_NORMAL_F64_DELTA=0), the table points that
    escape to the mirror, and the largest stored correction of r and c."""
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    idx = dev.index if dev.index is not None else torch.cuda.current_device()
    v = [C.c_uint64() for _ in range(5)]
    _lib.check(_lib.LIB.sdr_normal_delta_info(idx, *[C.byref(x) for x in v]), "sdr_normal_delta_info")
    return {"device_bytes": v[0].value, "escapes_r": v[1].value, "escapes_c": v[2].value,
            "max_abs_r": v[3].value, "max_abs_c": v[4].value}


def normal_fallback_count(device=None) -> int:
    idx = torch.cuda.current_device() if device is None else torch.device(device).index
    n = C.c_uint64()
    _lib.check(_lib.LIB.sdr_normal_fallback_count(idx, C.byref(n)), "sdr_normal_fallback_count")
    return int(n.value)


# ---------------------------------------------------------------------------
# Fills
# ---------------------------------------------------------------------------
def _param_error(status):
    if status == _lib.E_PARAM:
        return ValueError("distribution parameter out of domain")
    if status == _lib.E_DTYPE:
        return TypeError("dtype not supported for this distribution")
    return None


def _device(device) -> torch.device:
    if device is None:
        return torch.device("cuda", torch.cuda.current_device())
    dev = torch.device(device)
    if dev.type != "cuda":
        raise ValueError(f"RNG kernels run on CUDA devices only, got {dev}")
    return dev if dev.index is not None else torch.device("cuda", torch.cuda.current_device())


_alloc_counter = {"max_elements": 0, "enabled": False}


def _note_allocation(n: int):
    if _alloc_counter["enabled"] and n > _alloc_counter["max_elements"]:
        _alloc_counter["max_elements"] = n


class track_allocations:
    """Context manager recording the largest single RNG fill, in elements
    (reference rng.py:245-265)."""

    def __enter__(self):
        _alloc_counter["enabled"] = True
        _alloc_counter["max_elements"] = 0
        return _alloc_counter

    def __exit__(self, *exc):
        _alloc_counter["enabled"] = False
        return False


def fill_random(view: ShardView, state: RngState, dist: Distribution, dtype=np.float64,
                theta: int = 1, *, out: torch.Tensor | None = None, device=None) -> torch.Tensor:
    """Fill one window (reference rng.py:185-205).  `theta` (local thread count)
    cannot change values and is validated only.  Does not advance `state`."""
    if theta < 1:
        raise ValueError("local thread count must be >= 1")
    if not isinstance(dist, Distribution) or type(dist).native is Distribution.native:
        raise TypeError(f"{type(dist).__name__} has no sm_100a kernel (no CPU fallback)")
    code = dist.out_code(dtype_code(dtype))
    dev = _device(device if out is None else out.device)
    if out is None:
        out = torch.empty(view.local_shape, dtype=_TORCH_OF_CODE[code], device=dev)
    elif (tuple(out.shape) != view.local_shape or out.dtype != _TORCH_OF_CODE[code]
          or not out.is_contiguous()):
        raise ValueError("`out` must be a contiguous tensor of the window's shape and dtype")
    if dist.kind == _lib.NORMAL:
        with torch.cuda.device(dev):
            ensure_normal_tables(dev)
    nd, nr, nv = dist.native(), state.native(), view.to_native()
    with torch.cuda.device(dev):
        st = _lib.LIB.sdr_fill(out.data_ptr() if out.numel() else None, code, C.byref(nd),
                               C.byref(nr), C.byref(nv), _lib.stream_handle(dev))
    _lib.check(st, "sdr_fill", _param_error)
    _note_allocation(view.num_local_elements)
    return out


def generate_global(global_shape, state: RngState, dist: Distribution, dtype=np.float64,
                    *, device=None) -> torch.Tensor:
    """The full tensor on one device; advances state (reference rng.py:208-217)."""
    out = fill_random(full_view(tuple(global_shape)), state, dist, dtype=dtype, device=device)
    state.advance(math.prod(global_shape), dist.blocks_per_element)
    return out


def generate_distributed(spec: ShardSpec, global_shape, state: RngState, dist: Distribution,
                         dtype=np.float64, *, devices=None) -> dict:
    """Every mesh coordinate's shard in this process (the single-process form
    of reference rng.py:220-235); `devices` optionally maps coord -> device.
    Advances state once."""
    out = {}
    for coord in spec.mesh.iter_coords():
        view = local_shape_and_offset(spec, tuple(global_shape), coord)
        dev = None if devices is None else devices[coord]
        out[coord] = fill_random(view, state, dist, dtype=dtype, device=dev)
    state.advance(math.prod(global_shape), dist.blocks_per_element)
    return out


def generate_local(spec: ShardSpec, global_shape, state: RngState, dist: Distribution,
                   dtype=np.float64, coord=None, *, device=None) -> torch.Tensor:
    """The multi-process form: only this rank's shard (coord defaults to this
    process's torch.distributed rank in spec.mesh).  Advances state once, with
    no communication."""
    if coord is None:
        import torch.distributed as dist_mod
        rank = dist_mod.get_rank() if dist_mod.is_initialized() else 0
        coord = spec.mesh.coords_of_rank(rank)
    view = local_shape_and_offset(spec, tuple(global_shape), tuple(coord))
    out = fill_random(view, state, dist, dtype=dtype, device=device)
    state.advance(math.prod(global_shape), dist.blocks_per_element)
    return out


def dropout_mask_local(view: ShardView, state: RngState, p: float, dtype=np.float64,
                       *, device=None) -> torch.Tensor:
    """Keep-mask of dropout(p): 1 where the element survives
    (reference rng.py:238-242).  Does not advance state."""
    if not 0.0 <= p < 1.0:
        raise ValueError(f"dropout needs p in [0, 1), got {p}")
    return fill_random(view, state, Bernoulli(1.0 - p), dtype=dtype, device=device)


# ---------------------------------------------------------------------------
# Raw Philox (reference rng.py:34-82)
# ---------------------------------------------------------------------------
def _u64_tensor(x, dev):
    if isinstance(x, torch.Tensor):
        return x.to(device=dev).to(torch.int64)
    arr = np.asarray(x, dtype=np.uint64).view(np.int64)
    return torch.as_tensor(arr.copy(), device=dev)


def philox_blocks(seed: int, tau, beta, *, device=None) -> torch.Tensor:
    """Philox4x32-10 words for (tau, beta) arrays: int64 tensor [n, 4] holding
    the uint32 words, computed on the GPU."""
    dev = _device(device)
    t = _u64_tensor(tau, dev).reshape(-1).contiguous()
    b = _u64_tensor(beta, dev).reshape(-1).contiguous()
    if t.numel() != b.numel():
        raise ValueError("tau and beta must have the same number of elements")
    words = torch.empty((t.numel(), 4), dtype=torch.int32, device=dev)
    with torch.cuda.device(dev):
        st = _lib.LIB.sdr_philox_blocks(t.data_ptr(), b.data_ptr(), t.numel(),
                                        int(seed) & 0xFFFFFFFFFFFFFFFF, words.data_ptr(),
                                        _lib.stream_handle(dev))
    _lib.check(st, "sdr_philox_blocks")
    return words.to(torch.int64) & 0xFFFFFFFF


def philox_4x32_10(key_lo: int, key_hi: int, c0, c1, c2, c3):
    """Vectorised Philox-4x32-10 over counter lanes (uint32 arrays); returns the
    four output word arrays as NumPy uint32 (reference rng.py:34-59).  Runs on
    the GPU."""
    c = [np.asarray(x, dtype=np.uint64) for x in (c0, c1, c2, c3)]
    beta = c[0] | (c[1] << np.uint64(32))
    tau = c[2] | (c[3] << np.uint64(32))
    seed = (int(key_lo) & 0xFFFFFFFF) | ((int(key_hi) & 0xFFFFFFFF) << 32)
    w = philox_blocks(seed, tau.reshape(-1), beta.reshape(-1)).cpu().numpy().astype(np.uint32)
    shape = np.broadcast(*c).shape
    return tuple(w[:, i].reshape(shape) for i in range(4))


def backend_block(seed: int, tau_virtual: int, beta_virtual: int) -> tuple[int, int, int, int]:
    """One block for a single (seed, thread, offset) (reference rng.py:62-73)."""
    w = philox_blocks(seed, [tau_virtual], [beta_virtual])
    return tuple(int(x) for x in w[0].tolist())


def _words_tensor(w, dev) -> torch.Tensor:
    """uint32 Philox words (NumPy array, Python ints or a torch tensor holding
    the uint32 values) as a contiguous int32 CUDA tensor of the same bits."""
    if isinstance(w, torch.Tensor):
        if w.dtype in (torch.int32, torch.uint32):
            t = w.view(torch.int32) if w.dtype == torch.uint32 else w
        else:  # wrap the uint32 value into int32 two's complement explicitly
            t = w.to(torch.int64) & 0xFFFFFFFF
            t = (t - (t >= 2 ** 31).to(torch.int64) * 2 ** 32).to(torch.int32)
        return t.to(device=dev).contiguous()
    a = np.ascontiguousarray(np.asarray(w, dtype=np.uint32))
    return torch.from_numpy(a.view(np.int32).copy()).to(dev)


def transform_words(dist: Distribution, words, dtype=np.float64, *, device=None) -> torch.Tensor:
    """Distribution.transform (reference rng.py:104-182): the values of `dist`
    for Philox blocks given by their words, computed on the GPU by the same
    device transform the fill kernels use (sdr_transform).  `words` is the
    reference's 4-tuple (w0, w1, w2, w3) of uint32 arrays (NumPy or torch);
    words 2-3 are never read.  The result has w0's shape and the dtype the
    reference returns (e.g. float64 for Uniform01 of a non-float32 dtype)."""
    if not isinstance(dist, Distribution) or type(dist).native is Distribution.native:
        raise TypeError(f"{type(dist).__name__} has no sm_100a kernel (no CPU fallback)")
    if len(words) != 4:
        raise ValueError(f"expected the 4 words of a Philox block, got {len(words)}")
    dev = _device(device)
    w0, w1 = _words_tensor(words[0], dev), _words_tensor(words[1], dev)
    if tuple(w0.shape) != tuple(w1.shape):
        raise ValueError(f"word arrays differ in shape: {tuple(w0.shape)} vs {tuple(w1.shape)}")
    code = dist.out_code(dtype_code(dtype))
    out = torch.empty(w0.shape, dtype=_TORCH_OF_CODE[code], device=dev)
    if dist.kind == _lib.NORMAL:
        with torch.cuda.device(dev):
            ensure_normal_tables(dev)
    nd = dist.native()
    n = w0.numel()
    with torch.cuda.device(dev):
        st = _lib.LIB.sdr_transform(w0.data_ptr() if n else None, w1.data_ptr() if n else None, n,
                                    C.byref(nd), out.data_ptr() if n else None, code,
                                    _lib.stream_handle(dev))
    _lib.check(st, "sdr_transform", _param_error)
    return out
