"""Per-launch overhead: one event pair per kernel vs one pair around N back-to-back kernels."""
import os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2509_07003_b200 import ops, rng as R

st = R.RngState(20240817)
def batch(fn, n=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    torch.cuda._sleep(int(4e6))
    a.record()
    for _ in range(n): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / n
for n in (1 << 10, 1 << 20, 1 << 24):
    x = torch.randn(n, device="cuda", dtype=torch.bfloat16); y = torch.empty_like(x)
    print(f"n={n:9d} back-to-back: dropout {batch(lambda: ops.dropout_apply(x, 0.1, st, out=y))*1e3:7.2f} us | "
          f"copy {batch(lambda: y.copy_(x))*1e3:7.2f} us", flush=True)
# rotating buffers, 16.8M elements each, 8 pairs (537 MB) so no step hits L2
xs = [torch.randn(1 << 24, device="cuda", dtype=torch.bfloat16) for _ in range(8)]
ys = [torch.empty_like(t) for t in xs]
i = [0]
def rot():
    k = i[0] % 8; i[0] += 1
    ops.dropout_apply(xs[k], 0.1, st, out=ys[k])
print(f"16.8M rotating 8 buffers back-to-back: {batch(rot, 40)*1e3:7.2f} us", flush=True)
