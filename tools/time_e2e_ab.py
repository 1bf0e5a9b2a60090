"""A/B of the dropout_host pipeline geometry (blocks per call, staging buffers)
on cfg2 at P=1: K stream-ordered calls between one event pair, as bench.py's
e2e leg.  python tools/time_e2e_ab.py"""
import math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2509_07003_b200 import ops, rng as R
from paper_2509_07003_b200.placement import full_view

dev = torch.device("cuda", 0)
shape = (8, 4096, 4096)
x = torch.randn(shape, dtype=torch.bfloat16, generator=torch.Generator().manual_seed(0))
xh = x.pin_memory()
yhs = [torch.empty_like(xh).pin_memory() for _ in range(2)]
view = full_view(shape)
K = 10
for nbuf in (3, 4, 6):
    for chunks in (16, 32, 64):
        ops._PIPE_NBUF = nbuf
        st = R.RngState(1)
        for i in range(2):
            ops.dropout_host(xh, 0.1, st, view, out=yhs[i % 2], device=dev, sync=True)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(True), torch.cuda.Event(True)
        a.record()
        for i in range(K):
            ops.dropout_host(xh, 0.1, st, view, out=yhs[i % 2], device=dev, chunks=chunks, sync=False)
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / K
        print(f"nbuf {nbuf} chunks {chunks}: {ms:.3f} ms/step, {4 * math.prod(shape) / ms / 1e6:.1f} GB/s", flush=True)
