import os, sys, numpy as np, torch, statistics
sys.path.insert(0, os.getcwd())
from paper_2509_07003_b200 import rng as R
from paper_2509_07003_b200.placement import full_view
R.ensure_normal_tables()
st = R.RngState(5)
for dt, tdt in ((np.float64, torch.float64), (np.float32, torch.float32), ("float16", torch.float16), ("bfloat16", torch.bfloat16)):
    for dist, nm in ((R.Normal(0, 1), "normal"), (R.Uniform(-1, 1), "uniform")):
        t = torch.empty((4096, 4096), dtype=tdt, device="cuda")
        f = lambda: R.fill_random(full_view((4096, 4096)), st, dist, dt, out=t)
        for _ in range(3): f()
        torch.cuda.synchronize()
        ev = [(torch.cuda.Event(True), torch.cuda.Event(True)) for _ in range(10)]
        torch.cuda._sleep(int(5e6))
        for a, b in ev:
            a.record(); f(); b.record()
        torch.cuda.synchronize()
        ms = statistics.median(a.elapsed_time(b) for a, b in ev)
        print(f"{nm:8s} {str(tdt):15s} {ms*1e3:8.1f} us {t.numel()/ms/1e6:7.1f} G elem/s", flush=True)
