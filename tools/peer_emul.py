"""cfg5 through the peer transport with every rank of the DP2 x TP4 mesh
emulated as a CUDA stream of ONE GPU (bench.py --workload peer).

Each emulated rank owns a peer heap (sdr_peer_heap_alloc; one process, so no
IPC open is needed) and holds its TP shard of one LLaMA-3-8B layer (bf16).
A step is the fused S->R all-gather over the 4 DP fibers (pack -> barrier ->
gather pull) followed by the fused P->S reduce-scatter of same-shaped grads
(pack_scatter -> barrier -> reduce pull), all 8 ranks concurrently, ordered
only by the device barriers.  All ranks share one GPU's HBM, so the rate is
HBM-side (every rank's pack + pull bytes), not an NVLink rate.
"""
import ctypes as C

import numpy as np
import torch

from paper_2509_07003_b200 import _lib
from paper_2509_07003_b200.movers import CudaMover, Member, layout

D, FF, KV = 4096, 14336, 1024
# name: (global shape, placement on (dp, tp)) as in bench_extra's cfg5
LAYER = {"q": ((D, D), (1, 0)), "k": ((KV, D), (1, 0)), "v": ((KV, D), (1, 0)),
         "o": ((D, D), (0, 1)), "gate": ((FF, D), (1, 0)), "up": ((FF, D), (1, 0)),
         "down": ((D, FF), (0, 1)), "n1": ((D,), (0, None)), "n2": ((D,), (0, None))}


def _geom(shape, dim, P):
    E = shape[dim]
    outer = int(np.prod(shape[:dim])) if dim else 1
    inner = int(np.prod(shape[dim + 1:])) if dim + 1 < len(shape) else 1
    return E, -(-E // P), outer, inner


class Emulated:
    def __init__(self, dp=2, tp=4, half=160 << 20):
        self.dp, self.tp, self.half = dp, tp, half
        self.n = dp * tp
        self.bases = []
        for _ in range(self.n):
            b, h = C.c_void_p(), _lib.SdrIpcHandle()
            _lib.check(_lib.LIB.sdr_peer_heap_alloc(0, _lib.PEER_FLAG_BYTES + 2 * half, C.byref(b),
                                                     C.byref(h)), "heap")
            self.bases.append(b.value)
        self.streams = [torch.cuda.Stream() for _ in range(self.n)]
        self.epoch = [0] * self.n
        self.calls = [0] * self.n
        self.fiber = [[r % tp + tp * j for j in range(dp)] for r in range(self.n)]  # rank = tp*dp_i + tp_i
        self.plan = [self._plan(r) for r in range(self.n)]
        self.gathered = sum(m.tensor.numel() * 2 for m in self.plan[0]["recv"])

    def _plan(self, r):
        dp_i, tp_i = divmod(r, self.tp)
        send, recv, full, piece = [], [], [], []
        for shape, (dd, td) in LAYER.values():
            s = list(shape)
            if td is not None:  # TP shard first (even splits here)
                s[td] //= self.tp
            E, c, outer, inner = _geom(s, dd, self.dp)
            lo, hi = min(E, dp_i * c), min(E, dp_i * c + c)
            mine = list(s)
            mine[dd] = hi - lo
            send.append(Member(torch.randn(mine, device="cuda").bfloat16(), outer, hi - lo, inner, c))
            recv.append(Member(torch.empty(s, device="cuda", dtype=torch.bfloat16), outer, E, inner, c))
            full.append(Member(torch.randn(s, device="cuda").bfloat16(), outer, E, inner, c))
            piece.append(Member(torch.empty(mine, device="cuda", dtype=torch.bfloat16), outer, hi - lo,
                                inner, c))
        seg = layout(send)
        for a, b in zip(send, recv):
            b.seg_off = a.seg_off
        rseg = layout(full)
        for a, b in zip(full, piece):
            b.seg_off = a.seg_off
        return {"send": send, "recv": recv, "full": full, "piece": piece, "seg": seg, "rseg": rseg,
                "a": [CudaMover._arr(x) for x in (send, recv, full, piece)]}

    def _halves(self, r):
        h = self.calls[r] & 1
        self.calls[r] += 1
        off = _lib.PEER_FLAG_BYTES + h * self.half
        return (C.c_void_p * self.dp)(*[self.bases[q] + off for q in self.fiber[r]])

    def _barrier(self, r, st):
        self.epoch[r] += 1
        flags = (C.c_void_p * self.dp)(*[self.bases[q] for q in self.fiber[r]])
        _lib.check(_lib.LIB.sdr_peer_barrier(flags, self.fiber[r].index(r), self.dp, self.epoch[r],
                                             int(20e9), st), "barrier")

    def step(self):
        for r in range(self.n):
            st = self.streams[r].cuda_stream
            p = self.plan[r]
            me = self.fiber[r].index(r)
            a_send, a_recv, a_full, a_piece = p["a"]
            segs = self._halves(r)
            _lib.check(_lib.LIB.sdr_pack_local(a_send, len(p["send"]), segs[me], st), "pack")
            self._barrier(r, st)
            _lib.check(_lib.LIB.sdr_unpack_gathered_peers(a_recv, len(p["recv"]), segs, self.dp, st), "g")
            bufs = self._halves(r)
            _lib.check(_lib.LIB.sdr_pack_scatter(a_full, len(p["full"]), bufs[me], p["rseg"], self.dp, st),
                       "ps")
            self._barrier(r, st)
            _lib.check(_lib.LIB.sdr_reduce_scatter_peers(a_piece, len(p["piece"]), bufs, p["rseg"], self.dp,
                                                         me, _lib.BF16, st), "r")

    def hbm_bytes_per_step(self):
        """Algorithmic HBM bytes of one step, all ranks: AG pack (r+w shard) +
        gather pull (r+w gathered); RS pack (r+w full) + reduce pull (read dp
        pieces, write one)."""
        tot = 0
        for p in self.plan:
            shard = sum(m.tensor.numel() * 2 for m in p["send"])
            full = sum(m.tensor.numel() * 2 for m in p["full"])
            piece = sum(m.tensor.numel() * 2 for m in p["piece"])
            tot += 2 * shard + 2 * full + 2 * full + (self.dp + 1) * piece
        return tot

    def check(self):
        """Every rank's gathered tensors equal the fiber's shards, and its
        reduced piece equals the fiber's sum (bf16 adds in rank order)."""
        torch.cuda.synchronize()
        for r in range(self.n):
            p = self.plan[r]
            fib = [self.plan[q] for q in self.fiber[r]]
            me = self.fiber[r].index(r)
            for i, (shape, (dd, td)) in enumerate(LAYER.values()):
                want = torch.cat([f["send"][i].tensor for f in fib], dim=dd)
                if not torch.equal(p["recv"][i].tensor, want):
                    return False
                acc = fib[0]["full"][i].tensor.float()
                for f in fib[1:]:
                    acc = (acc + f["full"][i].tensor.float()).bfloat16().float()
                E, c, _, _ = _geom(list(p["full"][i].tensor.shape), dd, self.dp)
                lo, hi = min(E, me * c), min(E, me * c + c)
                if not torch.equal(p["piece"][i].tensor, acc.bfloat16().narrow(dd, lo, hi - lo)):
                    return False
        return True

    def close(self):
        torch.cuda.synchronize()
        for b in self.bases:
            _lib.LIB.sdr_peer_heap_free(b)
