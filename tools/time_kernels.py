"""Kernel timings for every BASELINE config on one GPU (CUDA events, launch
queue pre-filled so host overhead is hidden; median of reps).

    python tools/time_kernels.py            [SDR_LIB_PATH=<so> for A/B builds]
"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2509_07003_b200 import create_mesh, init as I, ops, rng as R
from paper_2509_07003_b200.placement import ShardSpec, full_view, local_shape_and_offset, parse_placements


def timeit(fn, reps=10, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(True), torch.cuda.Event(True)) for _ in range(reps)]
    # queue a ~reps ms spin first so the host overhead of fn() is hidden
    torch.cuda._sleep(int(2e6) * max(1, reps // 5))
    for a, b in ev:
        a.record()
        fn()
        b.record()
    torch.cuda.synchronize()
    return statistics.median(a.elapsed_time(b) for a, b in ev)


def line(name, ms, elems, bytes_):
    print(f"{name:48s} {ms*1e3:9.1f} us  {elems/ms/1e6:7.1f} G elem/s  {bytes_/ms/1e6:7.1f} GB/s", flush=True)


st = R.RngState(20240817)
# cfg2 dropout
x = torch.randn((8, 4096, 4096), device="cuda", dtype=torch.bfloat16)
y = torch.empty_like(x)
line("cfg2 dropout bf16 [8,4096,4096] P=1", timeit(lambda: ops.dropout_apply(x, 0.1, st, out=y)),
     x.numel(), x.numel() * 4)
mesh8 = create_mesh([("sp", 8)])
v = local_shape_and_offset(ShardSpec(mesh8, parse_placements("S(1)")), x.shape, (3,))
xs = x[:, v.local_offset[1]:v.local_offset[1] + v.local_shape[1]].contiguous()
ys = torch.empty_like(xs)
line("cfg2 dropout shard P=8", timeit(lambda: ops.dropout_apply(xs, 0.1, st, v, out=ys)), xs.numel(),
     xs.numel() * 4)
mk = torch.empty(x.shape, dtype=torch.uint8, device="cuda")
line("cfg2 dropout + uint8 mask out", timeit(lambda: ops.dropout_apply(x, 0.1, st, out=y, mask=mk)),
     x.numel(), x.numel() * 5)
del x, y, mk
# cfg1 randn f32 4096^2 (P=1 and P=2 shard)
for dt, nm in [(np.float32, "f32"), ("bfloat16", "bf16")]:
    t = torch.empty((4096, 4096), device="cuda", dtype=R.torch_dtype(dt))
    line(f"cfg1 normal {nm} [4096,4096]", timeit(lambda: R.fill_random(full_view((4096, 4096)), st, R.Normal(0, 1), dt, out=t)),
         t.numel(), t.numel() * t.element_size())
    line(f"uniform01 f32 [4096,4096]", timeit(lambda: R.fill_random(full_view((4096, 4096)), st, R.Uniform01(), np.float32,
                                                                       out=torch.empty((4096, 4096), device='cuda'))),
         t.numel(), t.numel() * 4) if nm == "f32" else None
print("normal fallbacks so far:", R.normal_fallback_count())
# cfg3 embedding on dp2 x tp4, rank (1,3), normal + uniform, f32 + bf16
mesh = create_mesh([("dp", 2), ("tp", 4)])
spec = ShardSpec(mesh, parse_placements("S(0),S(1)"))
v3 = local_shape_and_offset(spec, (50257, 4096), (0, 1))
b = 3 ** 0.5 * 0.02
for dist, dn in [(R.Normal(0, 0.02), "normal"), (R.Uniform(-b, b), "uniform")]:
    for dt in (np.float32, "bfloat16"):
        t = torch.empty(v3.local_shape, device="cuda", dtype=R.torch_dtype(dt))
        line(f"cfg3 {dn} {t.dtype} shard {v3.local_shape}", timeit(lambda: R.fill_random(v3, st, dist, dt, out=t)),
             t.numel(), t.numel() * t.element_size())
# cfg4 llama3-8b init, TP=8 shard (rank 0) and TP=1 (full), bf16, normal(0,0.02)
for tp in (8, 1):
    params = I.llama3_8b_params(lambda n, s: R.Normal(0.0, 0.02), "bfloat16")
    m = create_mesh([("tp", tp)])
    specs = I.llama3_tp_specs(params, m)
    n_el = sum(int(np.prod(local_shape_and_offset(specs[k], p.shape, (0,)).local_shape)) for k, p in params.items())

    def run():
        for p in params.values():
            p.value = None
        I.materialize(params, R.RngState(1234), specs, (0,))
    ms = timeit(run, reps=3, warm=1)
    line(f"cfg4 llama3-8b init normal bf16 TP={tp} (rank 0)", ms, n_el, n_el * 2)
    for p in params.values():
        p.value = None
    del params
    torch.cuda.empty_cache()
# cfg5 pack / unpack (HBM-bound copies around the coalesced NCCL call):
# one LLaMA-3-8B layer's 9 bf16 tensors on DP=2 (rank 0 shards), packed
# rank-major for a reduce-scatter and unpacked after an all-gather.
from paper_2509_07003_b200.movers import CudaMover, Member, layout
d, ff, kv = 4096, 14336, 1024
shapes = [((d, d), 1), ((kv, d), 1), ((kv, d), 1), ((d, d), 0), ((ff, d), 1), ((ff, d), 1), ((d, ff), 0),
          ((d,), 0), ((d,), 0)]
P = 2
fulls, full_m, loc_m = [], [], []
for shp, dim in shapes:
    f = torch.randn(shp, device="cuda", dtype=torch.bfloat16)
    outer, inner, rows = int(np.prod(shp[:dim])), int(np.prod(shp[dim + 1:])), shp[dim]
    chunk = -(-rows // P)
    full_m.append(Member(f, outer, rows, inner, chunk))
    loc = f.narrow(dim, 0, chunk).contiguous()
    loc_m.append(Member(loc, outer, chunk, inner, chunk))
seg = layout(full_m)
for a, b in zip(loc_m, full_m):
    a.seg_off = b.seg_off
mv = CudaMover()
packed = torch.empty(seg * P, dtype=torch.uint8, device="cuda")
nbytes = sum(m.tensor.numel() * 2 for m in full_m)
line("cfg5 pack_scatter (9 tensors, P=2)", timeit(lambda: mv.pack_scatter(full_m, packed, seg, P)), nbytes // 2,
     2 * nbytes)
line("cfg5 unpack_gathered (9 tensors, P=2)", timeit(lambda: mv.unpack_gathered(full_m, packed, seg, P)),
     nbytes // 2, 2 * nbytes)
segbuf = torch.empty(seg, dtype=torch.uint8, device="cuda")
line("cfg5 pack_local (9 shards)", timeit(lambda: mv.pack_local(loc_m, segbuf)), nbytes // 4, nbytes)
print("(pack rows: 'G elem/s' column = bf16 elements moved; GB/s = read + write bytes; HBM peak 6552 GB/s)")
