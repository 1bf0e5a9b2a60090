"""Dropout kernel time vs size and view (small-shard efficiency for strong scaling)."""
import os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2509_07003_b200 import create_mesh, ops, rng as R
from paper_2509_07003_b200.placement import ShardSpec, local_shape_and_offset, parse_placements
from tools.time_ab import timeit

st = R.RngState(20240817)
x = torch.randn((8, 4096, 4096), device="cuda", dtype=torch.bfloat16)
for P in (1, 2, 4, 8, 16):
    v = local_shape_and_offset(ShardSpec(create_mesh([("sp", P)]), parse_placements("S(1)")), x.shape, (P - 1,))
    xs = x[:, v.local_offset[1]:v.local_offset[1] + v.local_shape[1]].contiguous(); ys = torch.empty_like(xs)
    ms = timeit(lambda: ops.dropout_apply(xs, 0.1, st, v, out=ys))
    n = xs.numel()
    xc = x.view(-1)[:n].view(xs.shape); yc = torch.empty_like(xc)
    msc = timeit(lambda: ops.dropout_apply(xc, 0.1, st, out=yc))
    print(f"P={P:2d} n={n/1e6:6.1f}M shard-view {ms*1e3:7.1f} us ({n/ms/1e6:6.1f} G/s) | contiguous {msc*1e3:7.1f} us ({n/msc/1e6:6.1f} G/s)", flush=True)
# fixed per-launch overhead: small contiguous sizes, next to a torch copy of the same bytes
for n in (1 << 10, 1 << 16, 1 << 20, 1 << 22, 1 << 24):
    xc = x.view(-1)[:n]; yc = torch.empty_like(xc)
    msc = timeit(lambda: ops.dropout_apply(xc, 0.1, st, out=yc))
    mcp = timeit(lambda: yc.copy_(xc))
    print(f"n={n:9d} dropout {msc*1e3:7.2f} us | torch copy {mcp*1e3:7.2f} us", flush=True)
