"""Peer-transport protocol under real concurrency on one GPU.

The multi-process tests (test_redistribute_gloo.py) map peer heaps through
CUDA IPC, but processes sharing a GPU are time-sliced, so their kernels never
overlap.  Here P "ranks" live in ONE process, each with its own stream and
its own peer heap (sdr_peer_heap_alloc; same-process pointers need no IPC
open), and their pack / barrier / pull kernels run concurrently.  Iterations
alternate heap halves exactly as peer.PeerHeap does, with fresh data each
iteration, so a pull that read a half being re-packed (a broken double-buffer
argument) or a barrier that released early would show up as a wrong result.
"""

import ctypes as C

import pytest
import torch

pytestmark = pytest.mark.gpu


def _mk(t, outer, rows, inner, chunk, seg_off=0):
    from paper_2509_07003_b200.movers import Member
    return Member(t, outer, rows, inner, chunk, seg_off)


class _Ranks:
    def __init__(self, P, half):
        from paper_2509_07003_b200 import _lib
        self.L, self.P, self.half = _lib, P, half
        self.bases, self.epoch, self.calls = [], [0] * P, [0] * P
        for _ in range(P):
            b, h = C.c_void_p(), _lib.SdrIpcHandle()
            _lib.check(_lib.LIB.sdr_peer_heap_alloc(0, _lib.PEER_FLAG_BYTES + 2 * half, C.byref(b),
                                                     C.byref(h)), "alloc")
            self.bases.append(b.value)
        self.flags = (C.c_void_p * P)(*self.bases)
        self.streams = [torch.cuda.Stream() for _ in range(P)]

    def half_ptrs(self, r):
        h = self.calls[r] & 1
        self.calls[r] += 1
        off = self.L.PEER_FLAG_BYTES + h * self.half
        return (C.c_void_p * self.P)(*[b + off for b in self.bases])

    def barrier(self, r):
        self.epoch[r] += 1
        st = self.L.LIB.sdr_peer_barrier(self.flags, r, self.P, self.epoch[r], int(20e9),
                                         self.streams[r].cuda_stream)
        self.L.check(st, "barrier")

    def close(self):
        torch.cuda.synchronize()
        for b in self.bases:
            self.L.LIB.sdr_peer_heap_free(b)


@pytest.mark.parametrize("P,iters", [(4, 24), (8, 12)])
def test_concurrent_ranks_gather_and_reduce_scatter(P, iters):
    from paper_2509_07003_b200 import _lib
    from paper_2509_07003_b200.movers import CudaMover, layout
    torch.manual_seed(0)
    shapes = [((64, 96), 1), ((333, 40), 0), ((7,), 0), ((8, 50, 6), 1), ((1024, 1536), 0)]
    R = _Ranks(P, 16 << 20)
    # every iteration's inputs and outputs exist before any launch, so the
    # ranks' streams run all iterations back to back with no host sync and no
    # cross-stream dependency: only the peer barriers order them
    fulls = [[torch.randn(s, device="cuda") for s, _ in shapes] for _ in range(iters)]
    partials = [[[torch.randint(-8, 9, s, device="cuda").float() for s, _ in shapes]
                 for _ in range(P)] for _ in range(iters)]
    plan = []  # plan[it][r] = (send, recv, fm, pm)
    for it in range(iters):
        row = []
        for r in range(P):
            send, recv, fm, pm = [], [], [], []
            for i, ((shp, dim), f) in enumerate(zip(shapes, fulls[it])):
                E = shp[dim]
                c = -(-E // P)
                lo, hi = min(E, r * c), min(E, r * c + c)
                outer = int(torch.tensor(shp[:dim]).prod()) if dim else 1
                inner = int(torch.tensor(shp[dim + 1:]).prod()) if dim + 1 < len(shp) else 1
                loc = f.narrow(dim, lo, hi - lo).contiguous()
                send.append(_mk(loc, outer, hi - lo, inner, c))
                recv.append(_mk(torch.full_like(f, float("nan")), outer, E, inner, c))
                fm.append(_mk(partials[it][r][i], outer, E, inner, c))
                pm.append(_mk(torch.full_like(loc, float("nan")), outer, hi - lo, inner, c))
            seg = layout(send)
            for a, b in zip(send, recv):
                b.seg_off = a.seg_off
            rseg = layout(fm)
            for a, b in zip(fm, pm):
                b.seg_off = a.seg_off
            row.append((send, recv, fm, pm, seg, rseg))
        plan.append(row)
    torch.cuda.synchronize()
    try:
        for it in range(iters):
            for r in range(P):
                st = R.streams[r].cuda_stream
                send, recv, fm, pm, seg, rseg = plan[it][r]
                segs = R.half_ptrs(r)  # S -> R
                _lib.check(_lib.LIB.sdr_pack_local(CudaMover._arr(send), len(send), segs[r], st), "pack")
                R.barrier(r)
                _lib.check(_lib.LIB.sdr_unpack_gathered_peers(CudaMover._arr(recv), len(recv), segs, P,
                                                              st), "gpull")
                bufs = R.half_ptrs(r)  # P -> S
                _lib.check(_lib.LIB.sdr_pack_scatter(CudaMover._arr(fm), len(fm), bufs[r], rseg, P, st),
                           "pack_scatter")
                R.barrier(r)
                _lib.check(_lib.LIB.sdr_reduce_scatter_peers(CudaMover._arr(pm), len(pm), bufs, rseg, P,
                                                             r, _lib.F32, st), "rpull")
        torch.cuda.synchronize()
    finally:
        R.close()
    bad, n = [], 0
    for it in range(iters):
        sums = [sum(partials[it][q][i] for q in range(P)) for i in range(len(shapes))]
        for r in range(P):
            send, recv, fm, pm, _, _ = plan[it][r]
            for i, ((shp, dim), f) in enumerate(zip(shapes, fulls[it])):
                E = shp[dim]
                c = -(-E // P)
                lo, hi = min(E, r * c), min(E, r * c + c)
                n += 2
                if not torch.equal(recv[i].tensor, f):
                    bad.append(("gather", it, r, i))
                if not torch.equal(pm[i].tensor, sums[i].narrow(dim, lo, hi - lo)):
                    bad.append(("reduce", it, r, i))
    assert not bad, f"{len(bad)} of {n} results differ (first {bad[:5]})"
