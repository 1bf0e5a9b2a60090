"""Per-block timeline of ops.dropout_host (events on the H2D / compute / D2H streams)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2509_07003_b200 import ops, rng as R
xh = torch.randn((8, 4096, 4096), dtype=torch.bfloat16).pin_memory(); yh = torch.empty_like(xh).pin_memory()
st = R.RngState(20240817)
log = []
orig_copy = torch.Tensor.copy_
def rec(name):
    e = torch.cuda.Event(enable_timing=True); e.record(torch.cuda.current_stream()); log.append((name, e))
def patched_copy(self, src, non_blocking=False):
    kind = "h2d" if self.is_cuda and not src.is_cuda else ("d2h" if src.is_cuda and not self.is_cuda else "dd")
    rec(kind + "0"); r = orig_copy(self, src, non_blocking=non_blocking); rec(kind + "1"); return r
orig_apply = ops.dropout_apply
def patched_apply(*a, **k):
    rec("k0"); r = orig_apply(*a, **k); rec("k1"); return r
ops.dropout_host(xh, 0.1, st, out=yh)
torch.Tensor.copy_ = patched_copy; ops.dropout_apply = patched_apply
t0 = torch.cuda.Event(enable_timing=True); t0.record()
ops.dropout_host(xh, 0.1, st, out=yh)
torch.cuda.synchronize()
torch.Tensor.copy_ = orig_copy; ops.dropout_apply = orig_apply
rows = [(n, t0.elapsed_time(e)) for n, e in log]
for n, t in rows: print(f"{n:4s} {t:8.3f} ms")
