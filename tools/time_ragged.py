"""Fast vs generic fill/dropout paths: shard windows whose inner extent is / is not a multiple of 8."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from tools.time_ab import timeit
from paper_2509_07003_b200 import rng as R, ops, create_mesh
from paper_2509_07003_b200.placement import ShardSpec, local_shape_and_offset, parse_placements
st = R.RngState(3)
mesh = create_mesh([("tp", 2)])
spec = ShardSpec(mesh, parse_placements("S(1)"))
for shape in [(4096, 8192), (4096, 8194), (4096, 8198)]:
    v = local_shape_and_offset(spec, shape, (1,))
    n = v.num_local_elements
    row = []
    for dist, name, dt in [(R.Uniform01(), "uniform01 f32", np.float32), (R.Normal(0, 1), "normal f32", np.float32),
                           (R.Normal(0, 0.02), "normal bf16", "bfloat16")]:
        t = torch.empty(v.local_shape, device="cuda", dtype=R.torch_dtype(dt))
        ms = timeit(lambda: R.fill_random(v, st, dist, dt, out=t))
        row.append(f"{name} {n/ms/1e6:.0f}")
    x = torch.randn(v.local_shape, device="cuda", dtype=torch.bfloat16); y = torch.empty_like(x)
    ms = timeit(lambda: ops.dropout_apply(x, 0.1, st, v, out=y))
    row.append(f"dropout bf16 {n/ms/1e6:.0f}")
    print(f"{shape} S(1) rank 1 local {v.local_shape}: " + " | ".join(row) + "  (G elem/s)", flush=True)
