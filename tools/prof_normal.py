"""Launch the Normal fill kernels a few times (for ncu captures):
normal f32 [4096,4096] (cfg1) then normal bf16 [4096,4096] and uniform f32."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2509_07003_b200 import rng as R
from paper_2509_07003_b200.placement import full_view

R.ensure_normal_tables()
st = R.RngState(20240817)
which = sys.argv[1:] or ["f32", "bf16", "u32"]
for w in which:
    dt = {"f32": np.float32, "bf16": "bfloat16", "u32": np.float32}[w]
    dist = R.Uniform01() if w == "u32" else R.Normal(0.0, 1.0)
    t = torch.empty((4096, 4096), device="cuda", dtype=R.torch_dtype(dt))
    for _ in range(3):
        R.fill_random(full_view((4096, 4096)), st, dist, dt, out=t)
torch.cuda.synchronize()
print("ok")
