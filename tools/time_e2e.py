"""dropout_host end-to-end GB/s vs block count and staging depth (cfg2, pinned host)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2509_07003_b200 import ops, rng as R
xh = torch.randn((8, 4096, 4096), dtype=torch.bfloat16).pin_memory(); yh = torch.empty_like(xh).pin_memory()
st = R.RngState(20240817)
for nbuf in (3, 4):
    ops._PIPE_NBUF = nbuf
    for chunks in (16, 64, 128, 256, 512):
        ops.dropout_host(xh, 0.1, st, out=yh, chunks=chunks); torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(5): ops.dropout_host(xh, 0.1, st, out=yh, chunks=chunks)
        dt = (time.perf_counter() - t0) / 5
        print(f"nbuf={nbuf} chunks={chunks:3d}: {dt*1e3:6.2f} ms  {xh.numel()*4/dt/1e9:6.1f} GB/s", flush=True)
