"""Pack / unpack of coalesced collective buffers on the device.

`CudaMover` drives the sm_100a copy kernels of libsdrng.so (sdr_pack_local,
sdr_unpack_local, sdr_pack_scatter, sdr_unpack_gathered; include/sdrng.h).
The redistribute engine (dtensor.redistribute_many, comm.*_grad_reduce) only
talks to a mover, so its host logic can also be exercised in CPU multi-process
tests with a test-side mover (tests/cpu_mover.py) -- the product always uses
CudaMover and refuses non-CUDA tensors.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import torch

from . import _lib


@dataclass
class Member:
    """One tensor of a coalesced call, viewed as [outer, rows, inner] around the
    split dim; its rank-r piece is rows [r*chunk, min((r+1)*chunk, rows)),
    padded to `chunk` rows inside each rank segment at byte offset seg_off."""
    tensor: torch.Tensor
    outer: int
    rows: int
    inner: int
    chunk: int
    seg_off: int = 0

    @property
    def seg_bytes(self) -> int:
        return self.outer * self.chunk * self.inner * self.tensor.element_size()

    def native(self) -> _lib.SdrPackMember:
        m = _lib.SdrPackMember()
        m.data = self.tensor.data_ptr() if self.tensor.numel() else None
        m.outer, m.rows, m.inner = self.outer, self.rows, self.inner
        m.chunk_rows, m.seg_off = self.chunk, self.seg_off
        m.elem_bytes = self.tensor.element_size()
        return m


def layout(members: list[Member], align: int = 16) -> int:
    """Assign seg_off to every member (16 B aligned); returns segment bytes."""
    off = 0
    for m in members:
        m.seg_off = off
        off += -(-m.seg_bytes // align) * align
    return off


class CudaMover:
    name = "cuda"

    @staticmethod
    def _arr(members):
        for m in members:
            if m.tensor.numel() and not m.tensor.is_cuda:
                raise ValueError("CudaMover needs CUDA tensors (no CPU fallback)")
            if not m.tensor.is_contiguous():
                raise ValueError("members must be contiguous")
        arr = (_lib.SdrPackMember * max(1, len(members)))()
        for i, m in enumerate(members):
            arr[i] = m.native()
        return arr

    def _dev(self, buf: torch.Tensor):
        return buf.device

    def pack_local(self, members, seg: torch.Tensor):
        arr = self._arr(members)
        with torch.cuda.device(seg.device):
            st = _lib.LIB.sdr_pack_local(arr, len(members), seg.data_ptr(), _lib.stream_handle(seg.device))
        _lib.check(st, "sdr_pack_local")

    def unpack_local(self, members, seg: torch.Tensor):
        arr = self._arr(members)
        with torch.cuda.device(seg.device):
            st = _lib.LIB.sdr_unpack_local(arr, len(members), seg.data_ptr(), _lib.stream_handle(seg.device))
        _lib.check(st, "sdr_unpack_local")

    def pack_scatter(self, members, packed: torch.Tensor, seg_bytes: int, nranks: int):
        arr = self._arr(members)
        with torch.cuda.device(packed.device):
            st = _lib.LIB.sdr_pack_scatter(arr, len(members), packed.data_ptr(), seg_bytes, nranks,
                                           _lib.stream_handle(packed.device))
        _lib.check(st, "sdr_pack_scatter")

    def unpack_gathered(self, members, packed: torch.Tensor, seg_bytes: int, nranks: int):
        arr = self._arr(members)
        with torch.cuda.device(packed.device):
            st = _lib.LIB.sdr_unpack_gathered(arr, len(members), packed.data_ptr(), seg_bytes, nranks,
                                              _lib.stream_handle(packed.device))
        _lib.check(st, "sdr_unpack_gathered")


    def slice_local(self, full_members, piece_members, rank: int, nranks: int):
        """Rank `rank`'s ceil-block rows of each full member into its piece
        (Replicate -> Shard, dtensor.py:247-251)."""
        fa, pa = self._arr(full_members), self._arr(piece_members)
        dev = full_members[0].tensor.device
        with torch.cuda.device(dev):
            st = _lib.LIB.sdr_slice_local(fa, pa, len(full_members), rank, nranks, _lib.stream_handle(dev))
        _lib.check(st, "sdr_slice_local")


DEFAULT_MOVER = CudaMover()
