"""Test-only mover: the pack/unpack layout of libsdrng's copy kernels restated
with torch slicing on CPU tensors, so the redistribute engine's host logic
(grouping, fiber groups, rank-segment layout, collective sequence) can run in
world_size > 1 gloo tests without a GPU.  The product uses movers.CudaMover."""

import torch


def _rows(t, outer, rows, inner):
    return t.contiguous().view(torch.uint8).reshape(outer, rows * inner * t.element_size()) if t.numel() \
        else None


def _rank_rows(rows, chunk, r):
    lo = min(rows, r * chunk)
    return lo, min(rows, lo + chunk) - lo


class TorchCpuMover:
    name = "torch-cpu (tests only)"

    def pack_local(self, members, seg):
        for m in members:
            if m.tensor.numel() == 0:
                continue
            es = m.tensor.element_size()
            src = m.tensor.contiguous().view(torch.uint8).reshape(m.outer, m.rows * m.inner * es)
            dst = seg[m.seg_off:m.seg_off + m.seg_bytes].view(m.outer, m.chunk * m.inner * es)
            dst[:, :m.rows * m.inner * es] = src

    def unpack_local(self, members, seg):
        for m in members:
            if m.tensor.numel() == 0:
                continue
            es = m.tensor.element_size()
            src = seg[m.seg_off:m.seg_off + m.seg_bytes].view(m.outer, m.chunk * m.inner * es)
            m.tensor.view(torch.uint8).reshape(m.outer, m.rows * m.inner * es).copy_(
                src[:, :m.rows * m.inner * es])

    def pack_scatter(self, members, packed, seg_bytes, nranks):
        for m in members:
            if m.tensor.numel() == 0:
                continue
            es = m.tensor.element_size()
            full = m.tensor.contiguous().view(torch.uint8).reshape(m.outer, m.rows, m.inner * es)
            for r in range(nranks):
                lo, n = _rank_rows(m.rows, m.chunk, r)
                base = r * seg_bytes + m.seg_off
                dst = packed[base:base + m.seg_bytes].view(m.outer, m.chunk, m.inner * es)
                dst[:, :n] = full[:, lo:lo + n]

    def unpack_gathered(self, members, packed, seg_bytes, nranks):
        for m in members:
            if m.tensor.numel() == 0:
                continue
            es = m.tensor.element_size()
            full = m.tensor.view(torch.uint8).reshape(m.outer, m.rows, m.inner * es)
            for r in range(nranks):
                lo, n = _rank_rows(m.rows, m.chunk, r)
                base = r * seg_bytes + m.seg_off
                src = packed[base:base + m.seg_bytes].view(m.outer, m.chunk, m.inner * es)
                full[:, lo:lo + n] = src[:, :n]

    def slice_local(self, full_members, piece_members, rank, nranks):
        for f, q in zip(full_members, piece_members):
            if q.tensor.numel() == 0:
                continue
            es = f.tensor.element_size()
            lo, n = _rank_rows(f.rows, f.chunk, rank)
            src = f.tensor.contiguous().view(torch.uint8).reshape(f.outer, f.rows, f.inner * es)
            q.tensor.view(torch.uint8).reshape(f.outer, n, f.inner * es).copy_(src[:, lo:lo + n])
