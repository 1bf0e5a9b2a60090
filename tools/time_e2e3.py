"""e2e variant: copy-engine H2D of x blocks, the fused kernel writes y straight
into pinned host memory (PCIe posted writes, no D2H copy engine)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2509_07003_b200 import ops, rng as R
from paper_2509_07003_b200.placement import full_view
xh = torch.randn((8, 4096, 4096), dtype=torch.bfloat16).pin_memory(); yh = torch.empty_like(xh).pin_memory()
st = R.RngState(20240817)
n = xh.numel() * 2
view = full_view(tuple(xh.shape))
blocks = list(ops._host_blocks(tuple(xh.shape), view, 16))
cap = max(int(xh[ix].numel()) for ix, _ in blocks)
bufs = [torch.empty(cap, dtype=torch.bfloat16, device="cuda") for _ in range(3)]
sh, sc = torch.cuda.Stream(), torch.cuda.Stream()
def run():
    done = [None] * 3
    for i, (ix, sub) in enumerate(blocks):
        b = i % 3
        xs = xh[ix]
        xin = bufs[b][:xs.numel()].view(xs.shape)
        ev = torch.cuda.Event()
        with torch.cuda.stream(sh):
            if done[b] is not None:
                sh.wait_event(done[b])
            xin.copy_(xs, non_blocking=True)
            ev.record(sh)
        with torch.cuda.stream(sc):
            sc.wait_event(ev)
            ops.dropout_apply(xin, 0.1, st, sub, out=yh[ix])  # y -> pinned host memory directly
            e2 = torch.cuda.Event(); e2.record(sc); done[b] = e2
    sc.synchronize()
run()
t0 = time.perf_counter()
for _ in range(5): run()
dt = (time.perf_counter() - t0) / 5
print(f"H2D copy + kernel writes y to host: {dt*1e3:.2f} ms  {2*n/dt/1e9:.1f} GB/s", flush=True)
ref = ops.dropout_apply(xh.cuda(), 0.1, st).cpu()
print("bit-exact:", torch.equal(ref.view(torch.int16), yh.view(torch.int16)))
t0 = time.perf_counter()
for _ in range(5): ops.dropout_host(xh, 0.1, st, out=yh)
dt = (time.perf_counter() - t0) / 5
print(f"staged dropout_host: {dt*1e3:.2f} ms  {2*n/dt/1e9:.1f} GB/s", flush=True)
