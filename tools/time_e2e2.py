"""e2e pipeline diagnostics: per-stream busy spans of ops.dropout_host (cfg2)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2509_07003_b200 import ops, rng as R
xh = torch.randn((8, 4096, 4096), dtype=torch.bfloat16).pin_memory(); yh = torch.empty_like(xh).pin_memory()
st = R.RngState(20240817)
n = xh.numel() * 2
# 1) pure bidirectional copy pipeline of the same blocks, no kernel
xd = torch.empty_like(xh, device="cuda"); yd = torch.empty_like(xh, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def bidir(blocks):
    per = 8 // blocks if blocks <= 8 else None
    with torch.cuda.stream(s1):
        for b in range(8): xd[b].copy_(xh[b], non_blocking=True)
    with torch.cuda.stream(s2):
        for b in range(8): yh[b].copy_(yd[b], non_blocking=True)
    torch.cuda.synchronize()
bidir(8)
t0 = time.perf_counter()
for _ in range(5): bidir(8)
dt = (time.perf_counter() - t0) / 5
print(f"bidirectional 8x33.5MB copies, no deps: {dt*1e3:.2f} ms -> {2*n/dt/1e9:.1f} GB/s algorithmic-equivalent", flush=True)
for chunks in (4, 8, 16):
    ops.dropout_host(xh, 0.1, st, out=yh, chunks=chunks); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(5): ops.dropout_host(xh, 0.1, st, out=yh, chunks=chunks)
    dt = (time.perf_counter() - t0) / 5
    print(f"dropout_host chunks={chunks}: {dt*1e3:.2f} ms {2*n/dt/1e9:.1f} GB/s", flush=True)
# 2) same pipeline with the kernel replaced by nothing (copies + event chain only)
real = ops.dropout_apply
ops.dropout_apply = lambda x, p, state, view, out=None, out_dtype=None: out
for chunks in (8, 16):
    ops.dropout_host(xh, 0.1, st, out=yh, chunks=chunks); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(5): ops.dropout_host(xh, 0.1, st, out=yh, chunks=chunks)
    dt = (time.perf_counter() - t0) / 5
    print(f"pipeline without kernel chunks={chunks}: {dt*1e3:.2f} ms {2*n/dt/1e9:.1f} GB/s", flush=True)
ops.dropout_apply = real
# 3) host enqueue time of one call (no sync): how long the Python loop takes
import paper_2509_07003_b200.ops as O
t0 = time.perf_counter()
torch.cuda._sleep(int(2e7))
orig_sync = torch.cuda.Stream.synchronize
for chunks in (16,):
    t1 = time.perf_counter()
    ops.dropout_host(xh, 0.1, st, out=yh, chunks=chunks)
    print(f"dropout_host wall incl. sleep: {(time.perf_counter()-t1)*1e3:.2f} ms", flush=True)
