import os, sys
sys.path.insert(0, "/root/repo" if os.path.exists("/root/repo") else ".")
import numpy as np, torch
from tools.time_ab import timeit
from paper_2509_07003_b200 import rng as R
from paper_2509_07003_b200.placement import full_view
st = R.RngState(7)
b = 3 ** 0.5 * 0.02
tag = os.path.basename(os.environ.get("SDR_LIB_PATH", "default"))
out = []
for dt, name in [("bfloat16", "bf16"), (np.float16, "f16"), (np.float32, "f32")]:
    t = torch.empty((25129, 1024), device="cuda", dtype=R.torch_dtype(dt))
    v = full_view((25129, 1024))
    ms = timeit(lambda: R.fill_random(v, st, R.Uniform(-b, b), dt, out=t))
    out.append(f"uniform {name} {ms*1e3:.1f} us {t.numel()/ms/1e6:.1f} G/s")
print(tag + ": " + " | ".join(out), flush=True)
