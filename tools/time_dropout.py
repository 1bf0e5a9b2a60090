"""A/B timing of dropout kernel builds: SDR_LIB_PATH=<so> python tools/time_dropout.py
Times sdr_dropout on BASELINE cfg2 (bf16 [8,4096,4096], p=0.1, full view) with
CUDA events, median of 20 launches after 5 warm-ups; also a 1/8 shard (S(1), P=8)."""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2509_07003_b200 import ops, rng as R, create_mesh
from paper_2509_07003_b200.placement import ShardSpec, local_shape_and_offset, parse_placements

def timeit(fn, reps=20):
    for _ in range(5): fn()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(True), torch.cuda.Event(True)
        a.record(); fn(); b.record(); b.synchronize(); ts.append(a.elapsed_time(b))
    return statistics.median(ts)

shape = (8, 4096, 4096)
x = torch.randn(shape, device="cuda", dtype=torch.bfloat16)
y = torch.empty_like(x)
st = R.RngState(20240817)
ms = timeit(lambda: ops.dropout_apply(x, 0.1, st, out=y))
n = x.numel()
mesh = create_mesh([("sp", 8)]); spec = ShardSpec(mesh, parse_placements("S(1)"))
v = local_shape_and_offset(spec, shape, (3,))
xs = x[:, v.local_offset[1]:v.local_offset[1] + v.local_shape[1]].contiguous(); ys = torch.empty_like(xs)
ms8 = timeit(lambda: ops.dropout_apply(xs, 0.1, st, v, out=ys))
f32 = torch.empty(shape, device="cuda", dtype=torch.float32)
msn = timeit(lambda: R.fill_random(R.full_view(shape) if hasattr(R, "full_view") else None, st, R.Normal(0, 1), torch.float32, out=f32)) if False else float("nan")
print(f"{os.environ.get('SDR_LIB_PATH','default')}: full {ms*1e3:.1f} us {n/ms/1e6:.1f} G elem/s | shard/8 {ms8*1e3:.1f} us {xs.numel()/ms8/1e6:.1f} G elem/s")
