"""GPU parity of the one-launch deferred init (K3) and of the pack kernels.

materialize() must equal the reference's sequential walk (model.py:121-132:
generate_distributed / generate_global per parameter in definition order) bit
for bit, and leave the RngState at the same offset (test_plan.py:124-139).
"""

import numpy as np
import pytest
import torch

from conftest import bits
from oracle import rng_oracle as O

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    import paper_2509_07003_b200 as S
    from paper_2509_07003_b200 import init as I, rng as R
    from paper_2509_07003_b200.movers import CudaMover, Member, layout
    from paper_2509_07003_b200.placement import ShardSpec, local_shape_and_offset, parse_placements


def _small_llama(dist, dtype):
    shapes = [("embed", (131, 64))]
    for i in range(3):
        shapes += [(f"l{i}.q", (64, 64)), (f"l{i}.k", (16, 64)), (f"l{i}.o", (64, 64)),
                   (f"l{i}.down", (64, 96)), (f"l{i}.norm", (64,))]
    shapes += [("lm_head", (131, 64))]
    return {n: I.Parameter(s, dist, dtype) for n, s in shapes}


@pytest.mark.parametrize("dist,dt", [(lambda: R.Normal(0.0, 0.02), "bfloat16"),
                                     (lambda: R.Uniform(-0.0346, 0.0346), np.float32),
                                     (lambda: R.Normal(1.0, 2.0), np.float64)])
def test_materialize_equals_sequential_walk(dist, dt):
    mesh = S.create_mesh([("dp", 2), ("tp", 4)])
    for coord in [(0, 0), (1, 3), (0, 2)]:
        params = _small_llama(dist(), dt)
        specs = I.llama3_tp_specs(params, mesh, tp_dim=1)
        specs["embed"] = ShardSpec(mesh, parse_placements("S(0),S(1)"))  # 2-d, uneven rows
        del specs["l1.q"]                                               # one full-tensor init
        st = R.RngState(77, 5, 64)
        got = I.materialize(params, st, specs, coord)
        ref_state = R.RngState(77, 5, 64)
        for name, p in params.items():
            spec = specs.get(name)
            if spec is None:
                want = R.generate_global(p.shape, ref_state, p.dist, dt)
            else:
                view = local_shape_and_offset(spec, p.shape, coord)
                want = R.fill_random(view, ref_state, p.dist, dt)
                ref_state.advance(int(np.prod(p.shape)))
            assert torch.equal(bits(got[name]), bits(want)), (name, coord)
        assert st.offset == ref_state.offset


def test_materialize_oracle_spot_check():
    params = {"w": I.Parameter((300, 40), R.Normal(0.0, 0.02), np.float32),
              "b": I.Parameter((40,), R.Uniform(-1, 1), np.float32)}
    st = R.RngState(5)
    out = I.materialize(params, st)
    ref_w = O.fill_global((300, 40), 5, 0, 65536, "normal", (0.0, 0.02), np.float32)
    ref_b = O.fill_global((40,), 5, 1, 65536, "uniform", (-1, 1), np.float32)
    assert out["w"].cpu().numpy().tobytes() == ref_w.tobytes()
    assert out["b"].cpu().numpy().tobytes() == ref_b.tobytes()
    assert st.offset == 2


def test_cuda_pack_kernels_match_torch_layout():
    import sys, os
    sys.path.insert(0, os.path.dirname(__file__))
    from cpu_mover import TorchCpuMover
    gpu, cpu = CudaMover(), TorchCpuMover()
    g = torch.Generator().manual_seed(0)
    specs = [((5, 7, 3), 1, torch.float32), ((9, 4), 0, torch.bfloat16), ((2, 10), 1, torch.int64),
             ((7,), 0, torch.uint8), ((1, 3, 5), 2, torch.float16), ((12, 33), 1, torch.float64)]
    for P in (1, 2, 3, 4, 8):
        fulls = [torch.randint(-100, 100, shp, generator=g).to(dt) for shp, _, dt in specs]
        mem_full_c, mem_full_g, mem_loc_c, mem_loc_g, k = [], [], [], [], P // 2
        for (shp, d, dt), f in zip(specs, fulls):
            outer, inner, rows = int(np.prod(shp[:d])), int(np.prod(shp[d + 1:])), shp[d]
            chunk = -(-rows // P)
            lo = min(rows, k * chunk)
            n = min(rows, lo + chunk) - lo
            loc = f.narrow(d, lo, n).contiguous()
            mem_full_c.append(Member(f, outer, rows, inner, chunk))
            mem_full_g.append(Member(f.cuda(), outer, rows, inner, chunk))
            mem_loc_c.append(Member(loc, outer, n, inner, chunk))
            mem_loc_g.append(Member(loc.cuda(), outer, n, inner, chunk))
        seg = layout(mem_full_c)
        for a, b, c, dd in zip(mem_full_g, mem_loc_c, mem_loc_g, mem_full_c):
            a.seg_off = b.seg_off = c.seg_off = dd.seg_off
        # reduce-scatter input packing
        pc = torch.zeros(seg * P, dtype=torch.uint8)
        pg = torch.zeros(seg * P, dtype=torch.uint8, device="cuda")
        cpu.pack_scatter(mem_full_c, pc, seg, P)
        gpu.pack_scatter(mem_full_g, pg, seg, P)
        assert torch.equal(pc, pg.cpu())
        # gather: every rank's segment -> full tensors
        outs_c = [Member(torch.zeros_like(m.tensor), m.outer, m.rows, m.inner, m.chunk, m.seg_off)
                  for m in mem_full_c]
        outs_g = [Member(torch.zeros_like(m.tensor), m.outer, m.rows, m.inner, m.chunk, m.seg_off)
                  for m in mem_full_g]
        cpu.unpack_gathered(outs_c, pc, seg, P)
        gpu.unpack_gathered(outs_g, pg, seg, P)
        for a, b, f in zip(outs_c, outs_g, fulls):
            assert torch.equal(a.tensor, b.tensor.cpu()) and torch.equal(a.tensor, f)
        # local segment pack / unpack round trip
        sc = torch.zeros(seg, dtype=torch.uint8)
        sg = torch.zeros(seg, dtype=torch.uint8, device="cuda")
        cpu.pack_local(mem_loc_c, sc)
        gpu.pack_local(mem_loc_g, sg)
        assert torch.equal(sc, sg.cpu())
        back = [Member(torch.zeros_like(m.tensor), m.outer, m.rows, m.inner, m.chunk, m.seg_off)
                for m in mem_loc_g]
        gpu.unpack_local(back, sg)
        for a, m in zip(back, mem_loc_g):
            assert torch.equal(a.tensor, m.tensor)


def test_materialize_torch_module_on_meta_device():
    import torch.nn as nn
    with torch.device("meta"):
        model = nn.Sequential(nn.Linear(64, 96, bias=True), nn.ReLU(), nn.Linear(96, 32, bias=False))
    mesh = S.create_mesh([("tp", 4)])
    specs = {"0.weight": ShardSpec(mesh, parse_placements("S(0)")),
             "0.bias": ShardSpec(mesh, parse_placements("S(0)")),
             "2.weight": ShardSpec(mesh, parse_placements("S(1)"))}
    init_fn = lambda name, p: R.Normal(0.0, 1.0 / p.shape[-1] ** 0.5) if p.dim() == 2 else R.Uniform(-0.1, 0.1)
    st = R.RngState(3)
    meta = I.materialize_module(model, init_fn, st, specs, (2,))
    ref_st = R.RngState(3)
    for name, p in model.named_parameters():
        shape, spec = meta[name]
        v = local_shape_and_offset(spec, shape, (2,))
        want = R.fill_random(v, ref_st, init_fn(name, torch.empty(shape, device="meta")), torch.float32)
        ref_st.advance(int(np.prod(shape)))
        assert p.is_cuda and torch.equal(bits(p.data), bits(want)), name
    assert st.offset == ref_st.offset
    assert model[0].weight.shape == (24, 64) and model[2].weight.shape == (32, 24)


@pytest.mark.parametrize("kind", ["normal", "uniform"])
def test_cfg4_llama3_8b_tp8_shards_equal_tp1(kind):
    """BASELINE config 4 at full size: the whole LLaMA-3-8B init (291 params,
    8.03 G bf16 elements, one launch) on 1 GPU, then every TP=8 rank's shards
    (one launch per rank) equal the corresponding slices bit for bit, the
    RngState offsets agree, and oracle spot checks pin absolute values."""
    b = 3 ** 0.5 * 0.02
    fac = (lambda n, s: R.Normal(0.0, 0.02)) if kind == "normal" else (lambda n, s: R.Uniform(-b, b))
    full = I.llama3_8b_params(fac, "bfloat16")
    st1 = R.RngState(1234)
    out1 = I.materialize(full, st1)
    mesh = S.create_mesh([("tp", 8)])
    specs = I.llama3_tp_specs(full, mesh)
    for rank in (0, 3, 7):
        params = I.llama3_8b_params(fac, "bfloat16")
        st8 = R.RngState(1234)
        out8 = I.materialize(params, st8, specs, (rank,))
        assert st8.offset == st1.offset
        for name, p in params.items():
            v = local_shape_and_offset(specs[name], p.shape, (rank,))
            sl = tuple(slice(o, o + n) for o, n in zip(v.local_offset, v.local_shape))
            assert torch.equal(bits(out8[name]), bits(out1[name][sl])), (name, rank)
        del out8, params
    # absolute values: oracle windows of three parameters (first, middle, last)
    offs = np.cumsum([0] + [int(np.prod(p.shape)) // 65536 + (int(np.prod(p.shape)) % 65536 > 0)
                            for p in full.values()])
    names = list(full)
    params = (("normal", (0.0, 0.02)) if kind == "normal" else ("uniform", (-b, b)))
    for idx in (0, 150, 290):
        name, shape = names[idx], full[names[idx]].shape
        rows = np.array([0, 1, shape[0] - 1]) if len(shape) == 2 else None
        win = [rows, np.arange(0, 64)] if rows is not None else [np.arange(shape[0] - 64, shape[0])]
        ref = O.fill_window(shape, win, 1234, int(offs[idx]), 65536, params[0], params[1], _bf16())
        t = out1[name]
        if rows is not None:
            got = t[torch.as_tensor(rows, device=t.device)][:, :64]
        else:
            got = t[shape[0] - 64:]
        got = got.contiguous().cpu().view(torch.int16).numpy().view(np.uint16)
        assert got.tobytes() == np.ascontiguousarray(ref).view(np.uint16).tobytes(), name
    del out1
    torch.cuda.empty_cache()


def _bf16():
    import ml_dtypes
    return ml_dtypes.bfloat16


def test_pack_kernels_capture_in_cuda_graph():
    """Small calls pass the job table as a kernel parameter: pack/unpack of a
    layer's members is stream-capturable and replays to the eager result."""
    P = 2
    shapes = [((64, 48), 1), ((33, 16), 0), ((16,), 0)]
    full_m, outs = [], []
    for shp, dim in shapes:
        f = torch.randn(shp, device="cuda", dtype=torch.bfloat16)
        outer, inner, rows = int(np.prod(shp[:dim])), int(np.prod(shp[dim + 1:])), shp[dim]
        full_m.append(Member(f, outer, rows, inner, -(-rows // P)))
    seg = layout(full_m)
    mv = CudaMover()
    eager = torch.zeros(seg * P, dtype=torch.uint8, device="cuda")  # pad rows stay 0 in both
    mv.pack_scatter(full_m, eager, seg, P)
    packed = torch.zeros(seg * P, dtype=torch.uint8, device="cuda")
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            mv.pack_scatter(full_m, packed, seg, P)
    packed.zero_()
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(packed, eager)


@pytest.mark.parametrize("P", [2, 8])
def test_cfg5_full_layer_pack_round_trip(P):
    """BASELINE config 5 at full size: one LLaMA-3-8B layer's 9 bf16 tensors
    (q,k,v,gate,up split on dim 1; o,down on dim 0; the norms) packed
    rank-major for a reduce-scatter and unpacked after a gather reproduce the
    tensors bit for bit, and rank k's local segment equals its rank segment."""
    d, ff, kv = 4096, 14336, 1024
    shapes = [((d, d), 1), ((kv, d), 1), ((kv, d), 1), ((d, d), 0), ((ff, d), 1), ((ff, d), 1),
              ((d, ff), 0), ((d,), 0), ((d,), 0)]
    mv = CudaMover()
    full_m, fulls = [], []
    for shp, dim in shapes:
        f = torch.randint(-30000, 30000, shp, device="cuda", dtype=torch.int16).view(torch.bfloat16)
        outer, inner, rows = int(np.prod(shp[:dim])), int(np.prod(shp[dim + 1:])), shp[dim]
        full_m.append(Member(f, outer, rows, inner, -(-rows // P)))
        fulls.append(f)
    seg = layout(full_m)
    packed = torch.zeros(seg * P, dtype=torch.uint8, device="cuda")
    mv.pack_scatter(full_m, packed, seg, P)
    outs = [Member(torch.empty_like(m.tensor), m.outer, m.rows, m.inner, m.chunk, m.seg_off) for m in full_m]
    mv.unpack_gathered(outs, packed, seg, P)
    for o, f in zip(outs, fulls):
        assert torch.equal(o.tensor.view(torch.int16), f.view(torch.int16))
    k = P - 1
    locs = []
    for (shp, dim), m in zip(shapes, full_m):
        lo = min(m.rows, k * m.chunk)
        n = min(m.rows, lo + m.chunk) - lo
        locs.append(Member(m.tensor.narrow(dim, lo, n).contiguous(), m.outer, n, m.inner, m.chunk, m.seg_off))
    segbuf = torch.zeros(seg, dtype=torch.uint8, device="cuda")
    mv.pack_local(locs, segbuf)
    assert torch.equal(segbuf, packed[k * seg:(k + 1) * seg])


def test_parameter_materialize_global_and_sharded():
    """Parameter.materialize_global / materialize_sharded (model.py:36-46): a
    rank's shard equals its slice of the global init and both advance the
    state by the same amount."""
    mesh = S.create_mesh([("dp", 2), ("tp", 4)])
    spec = ShardSpec(mesh, parse_placements("S(0),S(1)"))
    p = I.Parameter((257, 64), R.Normal(0.0, 0.02), "bfloat16")
    sg = R.RngState(9, 2, 64)
    full = p.materialize_global(sg)
    for coord in [(0, 0), (1, 3)]:
        q = I.Parameter((257, 64), R.Normal(0.0, 0.02), "bfloat16")
        ss = R.RngState(9, 2, 64)
        d = q.materialize_sharded(spec, ss, coord)
        v = local_shape_and_offset(spec, (257, 64), coord)
        sl = tuple(slice(o, o + n) for o, n in zip(v.local_offset, v.local_shape))
        assert torch.equal(bits(d.local), bits(full[sl])) and ss.offset == sg.offset


def test_deferred_init_allocates_shard_sized_buffers():
    """Port of the reference's test_plan.py:124-139 onto init.materialize (the
    one-launch deferred init): with fc1.weight S(1) and fc2.weight S(0) on a
    4-rank tp mesh, every fill is shard-sized, and the merged shards equal the
    eager single-device init bitwise."""
    mesh = S.create_mesh([("tp", 4)])
    # MLP(16, 32, 8) of the reference: fc1 [16, 32], fc2 [32, 8], scaled-normal init (model.py:140-160)
    def params():
        return {"fc1.weight": I.Parameter((16, 32), R.Normal(0.0, 16 ** -0.5), np.float64),
                "fc2.weight": I.Parameter((32, 8), R.Normal(0.0, 32 ** -0.5), np.float64)}
    specs = {"fc1.weight": ShardSpec(mesh, parse_placements("S(1)")),
             "fc2.weight": ShardSpec(mesh, parse_placements("S(0)"))}
    shards = {}
    for coord in mesh.iter_coords():
        with R.track_allocations() as alloc:
            shards[coord] = I.materialize(params(), R.RngState(7), specs, coord)
        assert 0 < alloc["max_elements"] <= 16 * 32 // 4
    ref = params()
    with R.track_allocations() as alloc:
        I.materialize(ref, R.RngState(7))
    assert alloc["max_elements"] == 16 * 32  # the eager path fills whole tensors
    fc1 = torch.cat([shards[(k,)]["fc1.weight"] for k in range(4)], dim=1)
    fc2 = torch.cat([shards[(k,)]["fc2.weight"] for k in range(4)], dim=0)
    assert torch.equal(bits(fc1), bits(ref["fc1.weight"].value))
    assert torch.equal(bits(fc2), bits(ref["fc2.weight"].value))


def _mixed_params():
    """Every (distribution, dtype) family the reference's Module.materialize can
    meet (model.py:21-46): float weights, int / bool buffers; 30 RandInt
    members cross one descriptor-upload chunk (24)."""
    ps = {"w": I.Parameter((48, 40), R.Normal(0.0, 0.02), np.float32),
          "wd": I.Parameter((9, 33), R.Uniform(-0.5, 0.5), np.float64),
          "mask": I.Parameter((64, 17), R.Bernoulli(0.3), np.bool_),
          "mask8": I.Parameter((40, 8), R.Bernoulli(0.7), np.uint8),
          "ids32": I.Parameter((24, 16), R.RandInt(-3, 1000), np.int32)}
    for i in range(30):
        ps[f"ids{i}"] = I.Parameter((5 + i, 8), R.RandInt(-(1 << 40), 1 << 41), np.int64)
    return ps


def test_materialize_integer_and_bool_params():
    """sdr_fill_batch fills int / bool parameters (RandInt, Bernoulli) too, bit
    for bit equal to the sequential fill_random walk, sharded and unsharded."""
    mesh = S.create_mesh([("tp", 4)])
    for coord in [None, (1,), (3,)]:
        params = _mixed_params()
        specs = {} if coord is None else {n: ShardSpec(mesh, parse_placements("S(0)")) for n in params
                                          if n != "wd"}
        st = R.RngState(123, 0, 64)
        got = I.materialize(params, st, specs, coord)
        ref_state = R.RngState(123, 0, 64)
        for name, p in params.items():
            spec = specs.get(name)
            if spec is None:
                want = R.generate_global(p.shape, ref_state, p.dist, p.dtype)
            else:
                want = R.fill_random(local_shape_and_offset(spec, p.shape, coord), ref_state, p.dist, p.dtype)
                ref_state.advance(int(np.prod(p.shape)))
            assert got[name].dtype == want.dtype and torch.equal(bits(got[name]), bits(want)), (name, coord)
        assert st.offset == ref_state.offset
    # and against the oracle for one int and one bool member
    out = I.materialize({"a": I.Parameter((7, 9), R.RandInt(5, 77), np.int64),
                         "b": I.Parameter((13,), R.Bernoulli(0.25), np.bool_)}, R.RngState(9))
    ref_a = O.fill_global((7, 9), 9, 0, 65536, "randint", (5, 77), np.int64)
    ref_b = O.fill_global((13,), 9, 1, 65536, "bernoulli", (0.25,), np.bool_)
    assert out["a"].cpu().numpy().tobytes() == ref_a.tobytes()
    assert out["b"].cpu().numpy().tobytes() == ref_b.tobytes()


def test_materialize_captures_in_cuda_graph():
    """The batched init is stream-ordered end to end (descriptors as kernel
    parameters, stream-ordered allocation): captured once, a replay rewrites
    every parameter with the eager values."""
    mesh = S.create_mesh([("tp", 2)])
    specs = {n: ShardSpec(mesh, parse_placements("S(0)")) for n in _mixed_params()}
    eager = I.materialize(_mixed_params(), R.RngState(31), specs, (1,))
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):  # warm-up off the capture (tables, allocator)
        I.materialize(_mixed_params(), R.RngState(31), specs, (1,))
    torch.cuda.current_stream().wait_stream(side)
    g = torch.cuda.CUDAGraph()
    params = _mixed_params()
    with torch.cuda.graph(g):
        got = I.materialize(params, R.RngState(31), specs, (1,))
    for t in got.values():
        t.zero_()
    g.replay()
    torch.cuda.synchronize()
    for name in eager:
        assert torch.equal(bits(got[name]), bits(eager[name])), name


def test_materialize_bf16_normal_miss_queue_overflow(monkeypatch):
    """The batched bfloat16 Normal init resolves uncertified elements through
    the per-warp queue, flushed per tile.  With SDR_NORMAL_PATH=f64 every
    element misses the float32 path (the queue overflows into the inline
    path); with =exact every element takes the NumPy mirror: all three runs
    are bit-identical."""
    def params():
        return {f"w{i}": I.Parameter((300 + 7 * i, 520), R.Normal(0.5 * i, 0.02 + 0.1 * i), "bfloat16")
                for i in range(5)}
    R.ensure_normal_tables()
    outs = {}
    for path in (None, "f64", "exact"):
        if path is None:
            monkeypatch.delenv("SDR_NORMAL_PATH", raising=False)
        else:
            monkeypatch.setenv("SDR_NORMAL_PATH", path)
        outs[path] = I.materialize(params(), R.RngState(99))
    torch.cuda.synchronize()
    for name in outs[None]:
        assert torch.equal(bits(outs[None][name]), bits(outs["f64"][name])), name
        assert torch.equal(bits(outs[None][name]), bits(outs["exact"][name])), name
