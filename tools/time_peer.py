"""Pull kernels of the peer transport with LOCAL 'peer' buffers (one GPU):
cfg5 LLaMA-3-8B layer, bf16, P = 2 and 8.  The peers' halves are P separate
local allocations, so this measures the kernels against HBM, not NVLink.
  gather pull : read P*seg, write the full tensors (P*seg payload)
  reduce pull : read P x my segment (P*seg/P... = P*seg_mine), write my pieces
"""
import ctypes as C
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from tools.time_ab import timeit
from paper_2509_07003_b200 import _lib
from paper_2509_07003_b200.movers import CudaMover, Member, layout

d, ff, kv = 4096, 14336, 1024
shapes = [((d, d), 1), ((kv, d), 1), ((kv, d), 1), ((d, d), 0), ((ff, d), 1), ((ff, d), 1), ((d, ff), 0), ((d,), 0), ((d,), 0)]
st = lambda: _lib.stream_handle(torch.device("cuda"))
for P in (2, 8):
    full_m, piece_m = [], []
    for shp, dim in shapes:
        f = torch.randn(shp, device="cuda", dtype=torch.bfloat16)
        outer, inner, rows = int(np.prod(shp[:dim])), int(np.prod(shp[dim + 1:])), shp[dim]
        chunk = -(-rows // P)
        full_m.append(Member(f, outer, rows, inner, chunk))
        mine = min(rows, chunk)
        piece_m.append(Member(torch.empty(f.narrow(dim, 0, mine).shape, device="cuda", dtype=f.dtype), outer, mine, inner, chunk))
    seg = layout(full_m)
    for a, b in zip(piece_m, full_m):
        a.seg_off = b.seg_off
    full_bytes = sum(m.tensor.numel() * 2 for m in full_m)
    mine_bytes = sum(m.tensor.numel() * 2 for m in piece_m)
    segs = [torch.randint(0, 255, (seg,), dtype=torch.uint8, device="cuda") for _ in range(P)]
    packed = [torch.randint(0, 255, (seg * P,), dtype=torch.uint8, device="cuda") for _ in range(P)]
    seg_ptrs = (C.c_void_p * P)(*[s.data_ptr() for s in segs])
    pk_ptrs = (C.c_void_p * P)(*[s.data_ptr() for s in packed])
    arr_full = CudaMover._arr(full_m)
    arr_piece = CudaMover._arr(piece_m)
    def gather():
        _lib.check(_lib.LIB.sdr_unpack_gathered_peers(arr_full, len(full_m), seg_ptrs, P, st()), "g")
    def reduce():
        _lib.check(_lib.LIB.sdr_reduce_scatter_peers(arr_piece, len(piece_m), pk_ptrs, seg, P, 0, _lib.BF16, st()), "r")
    one = torch.empty(seg * P, dtype=torch.uint8, device="cuda")
    mv = CudaMover()
    out = []
    for n, f, b in [("gather_pull", gather, 2 * full_bytes),
                    ("reduce_pull", reduce, P * mine_bytes + mine_bytes),
                    ("unpack_gathered(local packed)", lambda: mv.unpack_gathered(full_m, one, seg, P), 2 * full_bytes)]:
        ms = timeit(f)
        out.append(f"{n} {ms*1e3:.1f} us {b/ms/1e6:.0f} GB/s")
    print(f"P={P}: " + " | ".join(out), flush=True)
# reference points: torch elementwise sums with the same read/write volume
for P in (2, 8):
    n = 218_103_808 // P  # my piece of the layer, bf16 elements
    xs = [torch.randn(n, device="cuda", dtype=torch.bfloat16) for _ in range(P)]
    z = torch.empty(n, device="cuda", dtype=torch.bfloat16)
    st_ = torch.stack(xs)
    def tsum():
        torch.sum(st_, dim=0, out=z)
    def tadd():
        torch.add(xs[0], xs[1], out=z)
    ms = timeit(tsum)
    b = (P + 1) * n * 2
    line = f"P={P}: torch.sum(stack) {ms*1e3:.1f} us {b/ms/1e6:.0f} GB/s"
    if P == 2:
        ms = timeit(tadd)
        line += f" | torch.add {ms*1e3:.1f} us {b/ms/1e6:.0f} GB/s"
    print(line, flush=True)
