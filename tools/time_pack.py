"""cfg5 pack/unpack copy kernels (A/B: SDR_LIB_PATH=variants/x.so)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from tools.time_ab import timeit
from paper_2509_07003_b200.movers import CudaMover, Member, layout
d, ff, kv = 4096, 14336, 1024
shapes = [((d, d), 1), ((kv, d), 1), ((kv, d), 1), ((d, d), 0), ((ff, d), 1), ((ff, d), 1), ((d, ff), 0), ((d,), 0), ((d,), 0)]
P = 2
full_m, loc_m = [], []
for shp, dim in shapes:
    f = torch.randn(shp, device="cuda", dtype=torch.bfloat16)
    outer, inner, rows = int(np.prod(shp[:dim])), int(np.prod(shp[dim + 1:])), shp[dim]
    chunk = -(-rows // P)
    full_m.append(Member(f, outer, rows, inner, chunk))
    loc_m.append(Member(f.narrow(dim, 0, chunk).contiguous(), outer, chunk, inner, chunk))
seg = layout(full_m)
for a, b in zip(loc_m, full_m):
    a.seg_off = b.seg_off
mv = CudaMover()
packed = torch.empty(seg * P, dtype=torch.uint8, device="cuda")
segbuf = torch.empty(seg, dtype=torch.uint8, device="cuda")
nbytes = sum(m.tensor.numel() * 2 for m in full_m)
tag = os.path.basename(os.environ.get("SDR_LIB_PATH", "default"))
r = [("pack_scatter", lambda: mv.pack_scatter(full_m, packed, seg, P), 2 * nbytes),
     ("unpack_gathered", lambda: mv.unpack_gathered(full_m, packed, seg, P), 2 * nbytes),
     ("pack_local", lambda: mv.pack_local(loc_m, segbuf), nbytes)]
out = []
for n, f, b in r:
    ms = timeit(f)
    out.append(f"{n} {ms*1e3:.1f} us {b/ms/1e6:.0f} GB/s")
src, dst = torch.empty(nbytes, dtype=torch.uint8, device="cuda"), torch.empty(nbytes, dtype=torch.uint8, device="cuda")
ms = timeit(lambda: dst.copy_(src))
out.append(f"torch copy {ms*1e3:.1f} us {2*nbytes/ms/1e6:.0f} GB/s")
print(tag + ": " + " | ".join(out), flush=True)
