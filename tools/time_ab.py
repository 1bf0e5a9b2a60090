"""A/B timing of library builds: SDR_LIB_PATH=<so> python tools/time_ab.py
Kernel time with CUDA events; a torch.cuda._sleep spin kernel is queued first so
the host enqueues every rep while the GPU is busy (no host gaps in the events)."""
import os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2509_07003_b200 import create_mesh, ops, rng as R
from paper_2509_07003_b200.placement import ShardSpec, full_view, local_shape_and_offset, parse_placements


def timeit(fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(True), torch.cuda.Event(True)) for _ in range(reps)]
    torch.cuda._sleep(int(2e6))  # ~1 ms spin: hides host launch overhead
    for a, b in ev:
        a.record(); fn(); b.record()
    torch.cuda.synchronize()
    return statistics.median(a.elapsed_time(b) for a, b in ev)


def main():
    tag = os.path.basename(os.environ.get("SDR_LIB_PATH", "default"))
    st = R.RngState(20240817)
    x = torch.randn((8, 4096, 4096), device="cuda", dtype=torch.bfloat16); y = torch.empty_like(x)
    ms = timeit(lambda: ops.dropout_apply(x, 0.1, st, out=y))
    v = local_shape_and_offset(ShardSpec(create_mesh([("sp", 8)]), parse_placements("S(1)")), x.shape, (3,))
    xs = x[:, v.local_offset[1]:v.local_offset[1] + v.local_shape[1]].contiguous(); ys = torch.empty_like(xs)
    ms8 = timeit(lambda: ops.dropout_apply(xs, 0.1, st, v, out=ys))
    t = torch.empty((4096, 4096), device="cuda")
    R.ensure_normal_tables()
    msn = timeit(lambda: R.fill_random(full_view((4096, 4096)), st, R.Normal(0, 1), np.float32, out=t))
    tb = torch.empty((4096, 4096), device="cuda", dtype=torch.bfloat16)
    msb = timeit(lambda: R.fill_random(full_view((4096, 4096)), st, R.Normal(0, 0.02), "bfloat16", out=tb))
    fb0 = R.normal_fallback_count()
    R.fill_random(full_view((4096, 4096)), st, R.Normal(0, 1), np.float32, out=t); torch.cuda.synchronize()
    fb1 = R.normal_fallback_count()
    R.fill_random(full_view((4096, 4096)), st, R.Normal(0, 0.02), "bfloat16", out=tb); torch.cuda.synchronize()
    fb2 = R.normal_fallback_count()
    print(f"{tag}: dropout full {ms*1e3:.1f} us ({x.numel()/ms/1e6:.1f} G/s) | dropout P=8 shard {ms8*1e3:.1f} us "
          f"({xs.numel()/ms8/1e6:.1f} G/s) | normal f32 4096^2 {msn*1e3:.1f} us ({t.numel()/msn/1e6:.1f} G/s) "
          f"| normal bf16 {msb*1e3:.1f} us ({tb.numel()/msb/1e6:.1f} G/s) | fallbacks/16.8M f32 {fb1-fb0} bf16 {fb2-fb1} "
          f"| calib {R._TABLE_ERRORS}", flush=True)


if __name__ == "__main__":
    main()
