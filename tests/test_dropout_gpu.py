"""GPU parity of the fused sharded dropout (mask + apply in one sm_100a kernel).

Reference semantics: ops.dropout (ops.py:168-190), dispatch dropout branch
(dispatch.py:567-576), dropout_mask_local (rng.py:238-242), k_dropout_apply
(engine.py:80-81); placement invariance (test_dispatch.py:183-193) and the
dropout gradient = rescaled mask (test_engine.py:86-95).
"""

import math

import numpy as np
import pytest
import torch

from conftest import bits, decode
from oracle import rng_oracle as O

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    import paper_2509_07003_b200 as S
    from paper_2509_07003_b200 import ops, rng as R
    from paper_2509_07003_b200.placement import ShardSpec, full_view, local_shape_and_offset, parse_placements

TORCH_DT = {"float32": torch.float32, "float64": torch.float64, "bfloat16": torch.bfloat16,
            "float16": torch.float16}


def test_golden_dropout(golden):
    man, arr = golden
    for c in man["dropout"]:
        x = decode(arr[c["key"] + "_x"], c["dtype"]).cuda()
        st = R.RngState(c["seed"], c["offset"], c["theta"])
        mask = torch.empty(x.shape, dtype=x.dtype, device="cuda")
        y_ref_dtype = torch.float32 if c["dtype"] == "bfloat16" else x.dtype
        y = ops.dropout_apply(x, c["p"], st, out_dtype=y_ref_dtype, mask=mask)
        assert torch.equal(bits(mask.cpu()), bits(decode(arr[c["key"] + "_mask"], c["dtype"])))
        assert torch.equal(bits(y.cpu()), bits(decode(arr[c["key"] + "_y"], c["y_dtype"]))), c
        if c["dtype"] == "bfloat16":  # torch-native bf16 output == ml_dtypes bf16 of the reference f32
            import ml_dtypes
            yb = ops.dropout_apply(x, c["p"], st)
            assert yb.dtype == torch.bfloat16
            ref16 = np.asarray(arr[c["key"] + "_y"]).astype(ml_dtypes.bfloat16)
            assert torch.equal(bits(yb.cpu()), bits(decode(ref16.view(np.uint16), "bfloat16")))
        # sharded masks are slices of the same draw
        mesh = S.create_mesh([("d", c["mesh"][0])])
        spec = ShardSpec(mesh, parse_placements(c["placements"]))
        for coord in mesh.iter_coords():
            v = local_shape_and_offset(spec, tuple(c["shape"]), coord)
            m = R.dropout_mask_local(v, st, c["p"], dtype=TORCH_DT[c["dtype"]])
            ref = decode(arr[c["key"] + "_mask_" + "_".join(map(str, coord))], c["dtype"]).reshape(m.shape)
            assert torch.equal(bits(m.cpu()), bits(ref))


@pytest.mark.parametrize("dt", ["float32", "bfloat16", "float16", "float64"])
@pytest.mark.parametrize("p", [0.1, 0.5, 0.999, 0.99999])  # 0.99999: float16 scale overflows to inf
def test_sharded_dropout_matches_oracle(dt, p):
    shape = (4, 96, 80)
    g = torch.Generator().manual_seed(5)
    x = torch.randn(shape, generator=g).to(TORCH_DT[dt]).cuda()
    specials = torch.tensor([float("nan"), float("inf"), -0.0, float("-inf"), -float("nan"), float("inf")],
                            dtype=x.dtype)
    x.view(-1)[:6] = specials
    x.view(-1)[100:106] = specials
    seed, off = 91, 12
    import ml_dtypes
    np_dt = ml_dtypes.bfloat16 if dt == "bfloat16" else np.dtype(dt)
    xn = x.cpu().view(torch.int16).numpy().view(np.uint16).view(ml_dtypes.bfloat16) if dt == "bfloat16" \
        else x.cpu().numpy()
    idx = [np.arange(n) for n in shape]
    m = O.keep_mask(shape, idx, seed, off, 65536, p, np_dt)
    yref = O.dropout_apply(xn, m, p)
    yref_t = torch.from_numpy(np.ascontiguousarray(yref))
    for P, pl in [(1, "S(1)"), (2, "S(1)"), (8, "S(1)"), (4, "S(2)"), (3, "S(0)")]:
        mesh = S.create_mesh([("sp", P)])
        spec = ShardSpec(mesh, parse_placements(pl))
        out_dtype = torch.float32 if dt == "bfloat16" else None
        for coord in mesh.iter_coords():
            v = local_shape_and_offset(spec, shape, coord)
            sl = tuple(slice(o, o + n) for o, n in zip(v.local_offset, v.local_shape))
            y = ops.dropout_apply(x[sl].contiguous(), p, R.RngState(seed, off), v, out_dtype=out_dtype)
            assert torch.equal(bits(y.cpu()), bits(yref_t[sl].contiguous())), (dt, p, pl, coord)
            if dt == "bfloat16":  # bf16 output = ml_dtypes' cast of the reference float32
                yb = ops.dropout_apply(x[sl].contiguous(), p, R.RngState(seed, off), v)
                r16 = np.ascontiguousarray(yref[sl]).astype(ml_dtypes.bfloat16).view(np.uint16)
                assert torch.equal(bits(yb.cpu()), bits(decode(r16, "bfloat16")))


def test_cfg2_full_size_sequence_parallel():
    """BASELINE config 2: x bf16 [8,4096,4096], p=0.1, Shard(1) over 1/2/4/8:
    shards (all 8 at P = 8) equal the slice of the unsharded result, and 512
    sequence rows (2 M elements, every batch, every P = 8 shard) equal the
    oracle."""
    shape = (8, 4096, 4096)
    x = torch.randn(shape, generator=torch.Generator(device="cuda").manual_seed(0), device="cuda",
                    dtype=torch.bfloat16)
    st = R.RngState(20240817)
    full = ops.dropout_apply(x, 0.1, st)
    for P in (2, 4, 8):
        mesh = S.create_mesh([("sp", P)])
        spec = ShardSpec(mesh, parse_placements("S(1)"))
        for coord in (mesh.iter_coords() if P == 8 else [(0,), (P - 1,)]):
            v = local_shape_and_offset(spec, shape, coord)
            s0, n = v.local_offset[1], v.local_shape[1]
            y = ops.dropout_apply(x[:, s0:s0 + n].contiguous(), 0.1, st, v)
            assert torch.equal(bits(y), bits(full[:, s0:s0 + n].contiguous()))
    import ml_dtypes
    # oracle rows: 64 sequence rows per batch spread over the whole sequence
    # (every Shard(1) rank at P = 8 owns 8 of them), all 8 batches: 2 M elements
    rows = np.linspace(0, 4095, 64).round().astype(np.int64)
    for b in range(8):
        xr = x[b, torch.from_numpy(rows).cuda()].cpu().view(torch.int16).numpy().view(np.uint16)
        xr = xr.view(ml_dtypes.bfloat16)
        j = ((b * 4096 + rows)[:, None] * 4096 + np.arange(4096)[None, :]).reshape(-1)
        keep = O.fill_indices(j, 20240817, 0, 65536, "bernoulli", (1.0 - 0.1,), ml_dtypes.bfloat16)
        yref = torch.from_numpy(O.dropout_apply(xr.reshape(-1), keep, 0.1)).to(torch.bfloat16)
        assert torch.equal(bits(full[b, torch.from_numpy(rows).cuda()].cpu().reshape(-1)), bits(yref)), b


def test_dropout_op_autograd_and_state():
    x = torch.randn(64, 33, device="cuda", requires_grad=True)
    st = R.RngState(3, 10, 64)
    y = ops.dropout(x, 0.25, state=st)
    assert st.offset == 10 + math.ceil(64 * 33 / 64)
    g = torch.randn_like(y)
    y.backward(g)
    mask = R.dropout_mask_local(full_view((64, 33)), R.RngState(3, 10, 64), 0.25, dtype=torch.float32)
    scale = np.float32(1 / (1 - 0.25))
    assert torch.equal(bits(x.grad), bits((g * mask) * scale))
    assert torch.equal(bits(y.detach()), bits((x.detach() * mask) * scale))
    st2 = R.RngState(3, 10, 64)
    assert ops.dropout(x, 0.0, state=st2) is x and st2.offset == 10


def test_dtensor_dropout_world_one():
    """DTensor-level dropout (dispatch.py:567-576) on a 1-rank mesh: same bits
    as the plain op, state advanced once."""
    from paper_2509_07003_b200.dtensor import from_local
    mesh = S.create_mesh([("d", 1)])
    spec = ShardSpec(mesh, parse_placements("S(0)"))
    x = torch.randn(16, 24, device="cuda")
    xd = from_local(x, spec, (16, 24), (0,))
    st = R.RngState(9)
    y = ops.dtensor_dropout(xd, 0.2, st)
    assert st.offset == 1
    ref = ops.dropout_apply(x, 0.2, R.RngState(9))
    assert torch.equal(bits(y.local), bits(ref))
    assert ops.dtensor_dropout(xd, 0.0, st) is xd and st.offset == 1


@pytest.mark.parametrize("dt,out_dtype", [(torch.bfloat16, None), (torch.bfloat16, torch.float32),
                                          (torch.float32, None)])
def test_dropout_host_pipeline_matches_device(dt, out_dtype):
    shape = (6, 37, 64)
    mesh = S.create_mesh([("sp", 3)])
    spec = ShardSpec(mesh, parse_placements("S(0)"))
    v = local_shape_and_offset(spec, (18, 37, 64), (1,))
    x = torch.randn(shape).to(dt).pin_memory()
    st = R.RngState(77, 4)
    for chunks in (1, 4, 6, 100):
        yh = ops.dropout_host(x, 0.3, st, v, out_dtype=out_dtype, chunks=chunks)
        yd = ops.dropout_apply(x.cuda(), 0.3, st, v, out_dtype=out_dtype)
        assert not yh.is_cuda and torch.equal(bits(yh), bits(yd.cpu())), chunks
    # Shard(1) window (sequence parallel), blocks split along dim 1
    v1 = local_shape_and_offset(ShardSpec(mesh, parse_placements("S(1)")), (6, 111, 64), (2,))
    for chunks in (3, 32):
        yh = ops.dropout_host(x, 0.3, st, v1, out_dtype=out_dtype, chunks=chunks)
        yd = ops.dropout_apply(x.cuda(), 0.3, st, v1, out_dtype=out_dtype)
        assert torch.equal(bits(yh), bits(yd.cpu())), chunks


@pytest.mark.parametrize("mask_dt", [torch.uint8, torch.bfloat16])
def test_ragged_rows_with_mask(mask_dt):
    """Windows whose rows are not a multiple of the 8-element chunk (chunked
    Philox, per-element I/O), with the mask output, vs the oracle."""
    import ml_dtypes
    shape, p, seed, off = (7, 101), 0.3, 123, 5
    x = torch.randn(shape, generator=torch.Generator().manual_seed(1)).to(torch.bfloat16).cuda()
    xn = x.cpu().view(torch.int16).numpy().view(np.uint16).view(ml_dtypes.bfloat16)
    m = O.keep_mask(shape, [np.arange(n) for n in shape], seed, off, 65536, p, ml_dtypes.bfloat16)
    yref = O.dropout_apply(xn, m, p)
    mesh = S.create_mesh([("tp", 3)])
    spec = ShardSpec(mesh, parse_placements("S(1)"))
    for coord in mesh.iter_coords():
        v = local_shape_and_offset(spec, shape, coord)  # 34 / 34 / 33 columns
        sl = tuple(slice(o, o + n) for o, n in zip(v.local_offset, v.local_shape))
        mask = torch.empty(v.local_shape, dtype=mask_dt, device="cuda")
        y = ops.dropout_apply(x[sl].contiguous(), p, R.RngState(seed, off), v, out_dtype=torch.float32,
                              mask=mask)
        assert torch.equal(bits(y.cpu()), bits(torch.from_numpy(np.ascontiguousarray(yref[sl])))), coord
        want = torch.from_numpy(np.ascontiguousarray(m[sl]).astype(np.float32))
        assert torch.equal(mask.float().cpu(), want), coord


def test_cuda_graph_capture_and_replay():
    """The fused kernels are stream-capturable: K dropout steps (each with its
    own RngState offset baked into its launch) and a Normal fill captured in
    one CUDA graph replay to exactly the eager results."""
    shape, p = (4, 256, 512), 0.1
    x = torch.randn(shape, device="cuda", dtype=torch.bfloat16)
    st = R.RngState(77)
    R.ensure_normal_tables()
    view = S.placement.full_view(shape)
    ys = [torch.empty_like(x) for _ in range(3)]
    w = torch.empty((300, 64), device="cuda")
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        ops.dropout_apply(x, p, st, view, out=ys[0])  # warm-up outside capture
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=s):
            cap = R.RngState(77)
            for y in ys:
                ops.dropout_apply(x, p, cap, view, out=y)
                cap.advance(x.numel())
            R.fill_random(S.placement.full_view((300, 64)), cap, R.Normal(0.0, 0.02), np.float32, out=w)
    for y in ys:
        y.zero_()
    w.zero_()
    g.replay()
    torch.cuda.synchronize()
    ref = R.RngState(77)
    for y in ys:
        assert torch.equal(bits(y), bits(ops.dropout_apply(x, p, ref, view)))
        ref.advance(x.numel())
    assert torch.equal(w, R.fill_random(S.placement.full_view((300, 64)), ref, R.Normal(0.0, 0.02), np.float32))


def test_dropout_host_async_back_to_back():
    """sync=False calls issued back to back (staging buffers reused across
    calls) give exactly the per-call results once the stream is drained."""
    shape, p = (8, 96, 64), 0.2
    x = torch.randn(shape).to(torch.bfloat16).pin_memory()
    outs = [torch.empty_like(x).pin_memory() for _ in range(5)]
    st = R.RngState(31)
    for i, o in enumerate(outs):
        ops.dropout_host(x, p, R.RngState(31, i), out=o, chunks=4, sync=False)
    torch.cuda.synchronize()
    for i, o in enumerate(outs):
        want = ops.dropout_apply(x.cuda(), p, R.RngState(31, i)).cpu()
        assert torch.equal(bits(o), bits(want)), i


def test_dropout_apply_rejects_bad_buffers():
    """A wrong `out` or `mask` must raise, never reach the kernel (a short or
    wrong-dtype buffer would be an out-of-bounds or wrong write)."""
    x = torch.randn(8, 64, device="cuda").to(torch.bfloat16)
    st = R.RngState(3)
    good = ops.dropout_apply(x, 0.1, st)
    for bad, exc in [(torch.empty(8, 64, device="cuda", dtype=torch.float16), TypeError),
                     (torch.empty(8, 63, device="cuda", dtype=torch.bfloat16), ValueError),
                     (torch.empty(64, 8, device="cuda", dtype=torch.bfloat16).t(), ValueError),
                     (torch.empty(8, 64, dtype=torch.bfloat16), ValueError)]:
        with pytest.raises(exc):
            ops.dropout_apply(x, 0.1, st, out=bad)
    for bad, exc in [(torch.empty(8, 64, dtype=torch.uint8), ValueError),        # host mask
                     (torch.empty(8, 32, device="cuda", dtype=torch.uint8), ValueError),
                     (torch.empty(8, 64, device="cuda", dtype=torch.int32), TypeError)]:
        with pytest.raises(exc):
            ops.dropout_apply(x, 0.1, st, mask=bad)
    with pytest.raises(TypeError):
        ops.dropout_apply(x, 0.1, st, out_dtype=torch.float16)
    y = torch.empty_like(x)
    m = torch.empty(8, 64, device="cuda", dtype=torch.bool)
    ops.dropout_apply(x, 0.1, st, out=y, mask=m)
    assert torch.equal(bits(y), bits(good))
    nz = x != 0
    assert torch.equal(m[nz], (good != 0)[nz])
