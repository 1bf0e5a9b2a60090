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


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16, torch.float16, torch.float64,
                                   torch.int32, torch.int64])
def test_pull_kernels_local_peers(dtype):
    """Both pull kernels with P local 'peer' buffers (no barrier): ragged
    members (odd extents, empty trailing pieces, 2-byte-aligned spans), every
    reducible dtype; sums of integer-valued data are exact in any order."""
    from paper_2509_07003_b200 import _lib
    from paper_2509_07003_b200.movers import CudaMover, layout
    code = {torch.float32: _lib.F32, torch.bfloat16: _lib.BF16, torch.float16: _lib.F16,
            torch.float64: _lib.F64, torch.int32: _lib.I32, torch.int64: _lib.I64}[dtype]
    g = torch.Generator(device="cuda").manual_seed(7)
    P = 5
    shapes = [((3, 17), 1), ((2,), 0), ((9, 4, 3), 1), ((40, 33), 0), ((1, 1), 0)]
    st = torch.cuda.current_stream().cuda_stream
    for r in range(P):
        fm, pm, want = [], [], []
        packed = []
        # every rank's full Partial tensor, packed rank-major by sdr_pack_scatter
        fulls = [[torch.randint(-50, 50, s, device="cuda", generator=g).to(dtype) for s, _ in shapes]
                 for _ in range(P)]
        for q in range(P):
            mq = []
            for (shp, dim), t in zip(shapes, fulls[q]):
                E = shp[dim]
                c = -(-E // P)
                outer = int(torch.tensor(shp[:dim]).prod()) if dim else 1
                inner = int(torch.tensor(shp[dim + 1:]).prod()) if dim + 1 < len(shp) else 1
                mq.append(_mk(t, outer, E, inner, c))
            seg = layout(mq)
            buf = torch.empty(seg * P, dtype=torch.uint8, device="cuda")
            _lib.check(_lib.LIB.sdr_pack_scatter(CudaMover._arr(mq), len(mq), buf.data_ptr(), seg, P, st), "ps")
            packed.append(buf)
            fm = mq
        for (shp, dim), m in zip(shapes, fm):
            E = shp[dim]
            c = -(-E // P)
            lo, hi = min(E, r * c), min(E, r * c + c)
            tot = sum(fulls[q][len(pm)] for q in range(P))
            want.append(tot.narrow(dim, lo, hi - lo))
            pm.append(_mk(torch.empty_like(want[-1]), m.outer, hi - lo, m.inner, c, m.seg_off))
        ptrs = (C.c_void_p * P)(*[b.data_ptr() for b in packed])
        _lib.check(_lib.LIB.sdr_reduce_scatter_peers(CudaMover._arr(pm), len(pm), ptrs, seg, P, r, code, st),
                   "rs")
        for w, m in zip(want, pm):
            assert torch.equal(m.tensor, w.to(dtype)), (dtype, r)
        # gather pull: segment q = rank q's shard, each in its own buffer
        segs, recv = [], []
        for q in range(P):
            sm = []
            for (shp, dim), t in zip(shapes, fulls[0]):
                E = shp[dim]
                c = -(-E // P)
                lo, hi = min(E, q * c), min(E, q * c + c)
                outer = int(torch.tensor(shp[:dim]).prod()) if dim else 1
                inner = int(torch.tensor(shp[dim + 1:]).prod()) if dim + 1 < len(shp) else 1
                sm.append(_mk(t.narrow(dim, lo, hi - lo).contiguous(), outer, hi - lo, inner, c))
            sseg = layout(sm)
            b = torch.empty(max(sseg, 16), dtype=torch.uint8, device="cuda")
            _lib.check(_lib.LIB.sdr_pack_local(CudaMover._arr(sm), len(sm), b.data_ptr(), st), "pl")
            segs.append(b)
            if q == 0:
                for (shp, dim), m in zip(shapes, sm):
                    recv.append(_mk(torch.empty(shp, dtype=dtype, device="cuda"), m.outer, shp[dim], m.inner,
                                    m.chunk, m.seg_off))
        sp = (C.c_void_p * P)(*[b.data_ptr() for b in segs])
        _lib.check(_lib.LIB.sdr_unpack_gathered_peers(CudaMover._arr(recv), len(recv), sp, P, st), "g")
        for m, t in zip(recv, fulls[0]):
            assert torch.equal(m.tensor, t), (dtype, "gather")


def test_cfg5_all_ranks_emulated_bit_exact():
    """cfg5 (DP2 x TP4, one LLaMA-3-8B layer, bf16): every rank's fused S->R
    and P->S through the peer transport, 8 ranks as concurrent streams, three
    back-to-back steps; gathered tensors exact, reduced pieces equal the
    rank-ordered bf16 sums."""
    import os
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from tools.peer_emul import Emulated
    em = Emulated()
    try:
        for _ in range(3):
            em.step()
        assert em.check()
    finally:
        em.close()
