"""Small workload for compute-sanitizer over the round-2 kernels: bfloat16
Normal fills through the per-warp miss queue (natural misses, and every
element missing with SDR_NORMAL_PATH=f64 in the environment, which also
overflows the queue), the batched init with its descriptor upload (mixed
dtypes, more members than one upload launch), checked against the exact path.
    compute-sanitizer --tool racecheck python tools/sanitize_r02.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2509_07003_b200 import init as I, rng as R
from paper_2509_07003_b200.placement import full_view

R.ensure_normal_tables()
st = R.RngState(7)
for shape in [(64, 256), (3, 1000, 8), (129, 72)]:
    t = R.fill_random(full_view(shape), st, R.Normal(0.0, 0.02), "bfloat16")
    torch.cuda.synchronize()
    assert torch.isfinite(t.float()).all()
ps = {f"w{i}": I.Parameter((33 + i, 40), R.Normal(0.0, 0.02), "bfloat16") for i in range(30)}
ps["ids"] = I.Parameter((17, 9), R.RandInt(0, 100), np.int64)
ps["mask"] = I.Parameter((5, 64), R.Bernoulli(0.5), np.bool_)
out = I.materialize(ps, R.RngState(3))
torch.cuda.synchronize()
print("sanitize workload ok", sum(v.numel() for v in out.values()))
