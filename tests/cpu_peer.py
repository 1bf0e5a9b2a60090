"""Test-only stand-in for peer.PeerHeap on CPU tensors: the same method
contract (all_gather / reduce_scatter / all_reduce over rank-segment layouts,
`half` capacity, regrowth on demand), with the bytes moved by gloo and the
reductions summed in ascending fiber-rank order.  Patched in for
peer.heap_for, it runs dtensor's peer-transport host logic -- bucketing by
heap half, regrow decisions, segment layouts, ledger entries -- in
world_size > 1 CPU tests.  The product path is peer.PeerHeap + csrc/peer.cu."""

import torch
import torch.distributed as dist

from cpu_mover import TorchCpuMover

_HEAPS = {}
LOG = []  # (kind, seg bytes) per pull, in call order


class GlooPeerHeap:
    def __init__(self, group, fiber, half):
        self.group, self.fiber, self.P = group, list(fiber), len(fiber)
        self.rank = self.fiber.index(dist.get_rank())
        self.half = int(half) // 256 * 256
        self.ok = True
        self.mv = TorchCpuMover()

    def all_gather(self, send, recv, seg):
        assert seg <= self.half
        buf = torch.zeros(seg, dtype=torch.uint8)
        self.mv.pack_local(send, buf)
        out = torch.empty(seg * self.P, dtype=torch.uint8)
        dist.all_gather_into_tensor(out, buf, group=self.group)
        self.mv.unpack_gathered(recv, out, seg, self.P)
        LOG.append(("all_gather", seg))

    def _ordered_sum(self, buf, dtype):
        parts = [torch.empty_like(buf) for _ in range(self.P)]
        dist.all_gather(parts, buf, group=self.group)
        acc = parts[0].view(dtype).clone()
        for p in parts[1:]:
            acc += p.view(dtype)
        return acc

    def reduce_scatter(self, full, piece, seg, dtype):
        assert seg * self.P <= self.half
        packed = torch.zeros(seg * self.P, dtype=torch.uint8)
        self.mv.pack_scatter(full, packed, seg, self.P)
        mine = packed.view(self.P, seg)
        sums = self._ordered_sum(mine.contiguous().view(-1), dtype).view(torch.uint8).view(self.P, seg)
        self.mv.unpack_local(piece, sums[self.rank].contiguous())
        LOG.append(("reduce_scatter", seg))

    def all_reduce(self, ins, outs):
        from paper_2509_07003_b200.movers import Member, layout
        full = [Member(t, 1, t.numel(), 1, -(-t.numel() // self.P)) for t in ins]
        seg = layout(full)
        if seg * (self.P + 1) > self.half:
            return False
        for t, o in zip(ins, outs):
            o.copy_(self._ordered_sum(t.contiguous().view(-1).view(torch.uint8), t.dtype).view(t.shape))
        LOG.append(("all_reduce", seg))
        return True


def heap_for(group, fiber, dev, need_half=0, initial_half=1 << 20, max_half=1 << 30):
    """peer.heap_for's contract on CPU: create on first use, regrow when a
    call needs a larger half (recorded in LOG as ('regrow', half))."""
    if group is None:
        return None
    key = tuple(fiber)
    hp = _HEAPS.get(key)
    need_half = -(-int(need_half) // 256) * 256
    if hp is None:
        hp = _HEAPS[key] = GlooPeerHeap(group, fiber, max(initial_half, min(need_half, max_half)))
    elif hp.half < need_half <= max_half:
        dist.barrier(group=group)
        hp = _HEAPS[key] = GlooPeerHeap(group, fiber, max(need_half, 2 * hp.half))
        LOG.append(("regrow", hp.half))
    return hp
