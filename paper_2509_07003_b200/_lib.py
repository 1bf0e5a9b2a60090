"""ctypes binding of the in-tree sm_100a C-ABI library `libsdrng.so`.

The declarations mirror include/sdrng.h one for one.  Importing this module
loads the library eagerly and raises if it is missing: there is no CPU
fallback anywhere in the product path.
"""

from __future__ import annotations

import ctypes as C
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SDR_LIB_PATH") or os.path.join(_HERE, "libsdrng.so")  # env: A/B kernel experiments

MAX_NDIM = 8

# sdr_status
OK, E_INVALID, E_DTYPE, E_DIST, E_PARAM, E_CUDA, E_NOTABLES, E_ALIGN = range(8)
# sdr_dtype
F32, F64, BF16, F16, I64, I32, U8, BOOL = range(8)
# sdr_dist_kind
UNIFORM01, UNIFORM, NORMAL, RANDINT, BERNOULLI = range(5)


class SdrDist(C.Structure):
    _fields_ = [("kind", C.c_int32), ("fparam", C.c_double * 2), ("iparam", C.c_int64 * 2)]


class SdrRng(C.Structure):
    _fields_ = [("seed", C.c_uint64), ("offset", C.c_uint64), ("theta", C.c_uint64)]


class SdrView(C.Structure):
    _fields_ = [
        ("ndim", C.c_int32),
        ("global_shape", C.c_int64 * MAX_NDIM),
        ("local_start", C.c_int64 * MAX_NDIM),
        ("local_len", C.c_int64 * MAX_NDIM),
        ("groups", C.c_int64 * MAX_NDIM),
        ("group_stride", C.c_int64 * MAX_NDIM),
    ]


class SdrPackMember(C.Structure):
    _fields_ = [
        ("data", C.c_void_p),
        ("outer", C.c_int64),
        ("rows", C.c_int64),
        ("inner", C.c_int64),
        ("chunk_rows", C.c_int64),
        ("seg_off", C.c_int64),
        ("elem_bytes", C.c_int32),
        ("pad_", C.c_int32),
    ]


MAX_PEERS = 64
PEER_FLAG_BYTES = 4096


class SdrIpcHandle(C.Structure):
    _fields_ = [("bytes", C.c_ubyte * 64)]


class NativeLibraryMissing(ImportError):
    pass


def _load():
    if not os.path.exists(LIB_PATH):
        raise NativeLibraryMissing(
            f"{LIB_PATH} not found: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(or `make -C paper_2509_07003_b200/csrc`). There is no CPU fallback.")
    lib = C.CDLL(LIB_PATH)
    P = C.POINTER
    sig = {
        "sdr_version": (C.c_int32, []),
        "sdr_strerror": (C.c_char_p, [C.c_int32]),
        "sdr_last_cuda_error": (C.c_char_p, []),
        "sdr_philox_block_host": (C.c_int32, [C.c_uint64, C.c_uint64, C.c_uint64, P(C.c_uint32)]),
        "sdr_philox_blocks": (C.c_int32, [C.c_void_p, C.c_void_p, C.c_int64, C.c_uint64,
                                          C.c_void_p, C.c_void_p]),
        "sdr_fill": (C.c_int32, [C.c_void_p, C.c_int32, P(SdrDist), P(SdrRng), P(SdrView),
                                 C.c_void_p]),
        "sdr_transform": (C.c_int32, [C.c_void_p, C.c_void_p, C.c_int64, P(SdrDist), C.c_void_p,
                                      C.c_int32, C.c_void_p]),
        "sdr_fill_batch": (C.c_int32, [P(C.c_void_p), P(C.c_int32), P(SdrDist), P(SdrRng),
                                       P(SdrView), C.c_int32, C.c_void_p]),
        "sdr_dropout": (C.c_int32, [C.c_void_p, C.c_int32, C.c_void_p, C.c_int32, C.c_void_p,
                                    C.c_int32, C.c_double, P(SdrRng), P(SdrView), C.c_void_p]),
        "sdr_normal_tables_load": (C.c_int32, [C.c_int32, C.c_void_p, C.c_void_p,
                                               P(C.c_double), P(C.c_double)]),
        "sdr_normal_tables_loaded": (C.c_int32, [C.c_int32]),
        "sdr_normal_delta_info": (C.c_int32, [C.c_int32] + [P(C.c_uint64)] * 5),
        "sdr_normal_mirror_info": (C.c_int32, [C.c_int32, P(C.c_uint64), P(C.c_uint64), P(C.c_int32),
                                               P(C.c_double)]),
        "sdr_normal_fallback_count": (C.c_int32, [C.c_int32, P(C.c_uint64)]),
        "sdr_unpack_gathered": (C.c_int32, [P(SdrPackMember), C.c_int32, C.c_void_p, C.c_int64,
                                            C.c_int32, C.c_void_p]),
        "sdr_pack_scatter": (C.c_int32, [P(SdrPackMember), C.c_int32, C.c_void_p, C.c_int64,
                                         C.c_int32, C.c_void_p]),
        "sdr_pack_local": (C.c_int32, [P(SdrPackMember), C.c_int32, C.c_void_p, C.c_void_p]),
        "sdr_unpack_local": (C.c_int32, [P(SdrPackMember), C.c_int32, C.c_void_p, C.c_void_p]),
        "sdr_slice_local": (C.c_int32, [P(SdrPackMember), P(SdrPackMember), C.c_int32, C.c_int32, C.c_int32,
                                        C.c_void_p]),
        "sdr_probe_int32": (C.c_int32, [C.c_int32, P(C.c_double), P(C.c_double), P(C.c_double)]),
        "sdr_peer_heap_alloc": (C.c_int32, [C.c_int32, C.c_int64, P(C.c_void_p), P(SdrIpcHandle)]),
        "sdr_peer_heap_open": (C.c_int32, [C.c_int32, P(SdrIpcHandle), P(C.c_void_p)]),
        "sdr_peer_heap_close": (C.c_int32, [C.c_void_p]),
        "sdr_peer_heap_free": (C.c_int32, [C.c_void_p]),
        "sdr_peer_barrier": (C.c_int32, [P(C.c_void_p), C.c_int32, C.c_int32, C.c_uint64, C.c_int64,
                                         C.c_void_p]),
        "sdr_peer_flag_read": (C.c_int32, [C.c_void_p, C.c_int32, P(C.c_uint64)]),
        "sdr_unpack_gathered_peers": (C.c_int32, [P(SdrPackMember), C.c_int32, P(C.c_void_p),
                                                  C.c_int32, C.c_void_p]),
        "sdr_reduce_scatter_peers": (C.c_int32, [P(SdrPackMember), C.c_int32, P(C.c_void_p),
                                                 C.c_int64, C.c_int32, C.c_int32, C.c_int32,
                                                 C.c_void_p]),
        "sdr_peer_all_gather": (C.c_int32, [P(SdrPackMember), P(SdrPackMember), C.c_int32, P(C.c_void_p),
                                            C.c_int32, C.c_int32, C.c_int64, C.c_uint64, C.c_int64,
                                            C.c_int32, C.c_void_p]),
        "sdr_peer_reduce_scatter": (C.c_int32, [P(SdrPackMember), P(SdrPackMember), C.c_int32,
                                                P(C.c_void_p), C.c_int32, C.c_int32, C.c_int64, C.c_int64,
                                                C.c_int32, C.c_uint64, C.c_int64, C.c_int32, C.c_void_p]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


LIB = _load()

EXPORTED = (
    "sdr_version", "sdr_strerror", "sdr_last_cuda_error", "sdr_philox_block_host",
    "sdr_philox_blocks", "sdr_fill", "sdr_transform", "sdr_fill_batch", "sdr_dropout", "sdr_normal_tables_load",
    "sdr_normal_tables_loaded", "sdr_normal_mirror_info", "sdr_normal_delta_info", "sdr_normal_fallback_count", "sdr_unpack_gathered",
    "sdr_pack_scatter", "sdr_pack_local", "sdr_unpack_local", "sdr_slice_local", "sdr_probe_int32",
    "sdr_peer_heap_alloc", "sdr_peer_heap_open", "sdr_peer_heap_close", "sdr_peer_heap_free",
    "sdr_peer_barrier", "sdr_peer_flag_read", "sdr_unpack_gathered_peers", "sdr_reduce_scatter_peers",
    "sdr_peer_all_gather", "sdr_peer_reduce_scatter",
)


class SdrError(RuntimeError):
    def __init__(self, status: int, what: str):
        msg = LIB.sdr_strerror(status).decode()
        if status == E_CUDA:
            msg += ": " + LIB.sdr_last_cuda_error().decode()
        super().__init__(f"{what}: {msg} (status {status})")
        self.status = status


def check(status: int, what: str, exc=None):
    """Map a nonzero sdr_status to an exception; `exc(status)` may pick the
    reference's exception type (ValueError for E_PARAM, etc.)."""
    if status == OK:
        return
    if exc is not None:
        e = exc(status)
        if e is not None:
            raise e
    raise SdrError(status, what)


def stream_handle(device: torch.device | None = None) -> int:
    """cudaStream_t of torch's current stream on `device`, as an int."""
    return torch.cuda.current_stream(device).cuda_stream
