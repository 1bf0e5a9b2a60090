import os, sys, time, cProfile, pstats
sys.path.insert(0, os.getcwd())
import torch
from paper_2509_07003_b200 import init as I, rng as R
params = I.llama3_8b_params(lambda nm, s: R.Normal(0.0, 0.02), "bfloat16")
from paper_2509_07003_b200 import create_mesh
mesh = create_mesh([("tp", 1)]); specs = I.llama3_tp_specs(params, mesh)
dev = torch.device("cuda", 0)
def step():
    for p in params.values(): p.value = None
    I.materialize(params, R.RngState(1), specs, (0,), device=dev)
for _ in range(2): step()
torch.cuda.synchronize()
t = time.perf_counter(); step(); h = time.perf_counter() - t; torch.cuda.synchronize(); tot = time.perf_counter() - t
print(f"host {h*1e3:.2f} ms, host+gpu {tot*1e3:.2f} ms")
pr = cProfile.Profile(); pr.enable(); step(); pr.disable(); torch.cuda.synchronize()
pstats.Stats(pr).sort_stats("cumtime").print_stats(12)
