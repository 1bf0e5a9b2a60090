"""Multi-process (gloo, CPU) tests of the redistribute engine's host logic:
fiber process groups, rank-segment layout with uneven (padded) shards,
multi-tensor coalescing, bucketed / N-d fused gradient reduction.

The reference's simulator results (tests/golden, produced by running
spmdsim.dtensor.redistribute) are the expected values; integer-valued data
makes every reduction order-independent, hence bit-exact (test_comm.py:46-58).
The pack/unpack step uses tests/cpu_mover.py (the GPU runs use the CUDA mover).
"""

import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

HERE = os.path.dirname(os.path.abspath(__file__))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _spawn(fn, ws, *args):
    port = _free_port()
    mp.spawn(_entry, args=(ws, port, fn, args), nprocs=ws, join=True)


def _entry(rank, ws, port, fn, args):
    sys.path[:0] = [HERE, os.path.dirname(HERE)]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    try:
        fn(rank, ws, *args)
    finally:
        dist.barrier()
        dist.destroy_process_group()


def _golden():
    import json
    with open(os.path.join(HERE, "golden", "manifest.json")) as f:
        man = json.load(f)
    return man, np.load(os.path.join(HERE, "golden", "golden.npz"))


def _worker_golden(rank, ws, mesh_sizes, bucket_bytes=None):
    from cpu_mover import TorchCpuMover
    from paper_2509_07003_b200 import dtensor as DT
    if bucket_bytes is not None:
        DT.PIPELINE_BUCKET_BYTES = bucket_bytes
    from paper_2509_07003_b200 import comm, create_mesh
    from paper_2509_07003_b200.dtensor import from_local, redistribute, redistribute_many
    from paper_2509_07003_b200.placement import ShardSpec, parse_placements
    man, arr = _golden()
    mover = TorchCpuMover()
    mesh = create_mesh([(f"m{j}", s) for j, s in enumerate(mesh_sizes)])
    coord = mesh.coords_of_rank(rank)
    tag = "_".join(map(str, coord))
    cases = [c for c in man["redistribute"] if tuple(c["mesh"]) == tuple(mesh_sizes)]
    assert cases
    xs, dsts, wants = [], [], []
    for c in cases:
        src = ShardSpec(mesh, parse_placements(c["src"]))
        dst = ShardSpec(mesh, parse_placements(c["dst"]))
        loc = torch.from_numpy(np.ascontiguousarray(arr[c["key"] + "_in_" + tag]))
        x = from_local(loc, src, tuple(c["shape"]), coord)
        ledger = comm.CollectiveLedger()
        y = redistribute(x, dst, ledger, mover=mover)
        want = arr[c["key"] + "_out_" + tag]
        assert y.local.numpy().tobytes() == np.ascontiguousarray(want).tobytes(), (c, coord)
        assert y.meta.spec == dst
        xs.append(x)
        dsts.append(dst)
        wants.append(want)
    # all cases of this mesh at once: coalesced into one collective per kind
    ledger = comm.CollectiveLedger()
    ys = redistribute_many(xs, dsts, ledger, mover=mover)
    for y, want, c in zip(ys, wants, cases):
        assert y.local.numpy().tobytes() == np.ascontiguousarray(want).tobytes(), ("many", c)
    per_dim_kinds = len(ledger.entries)
    if bucket_bytes is None:  # one coalesced collective per (dim, kind)
        assert per_dim_kinds <= 3 * len(mesh_sizes), ledger.entries
    elif bucket_bytes == 1:  # one collective per member
        assert per_dim_kinds >= len(cases), ledger.entries


@pytest.mark.parametrize("mesh_sizes", [(4,), (2,), (2, 4)])
def test_redistribute_matches_reference_golden(mesh_sizes):
    _spawn(_worker_golden, int(np.prod(mesh_sizes)), mesh_sizes)


def test_redistribute_many_bucketed_pipeline_golden():
    """One member per bucket (the pipelined path) still reproduces the reference."""
    _spawn(_worker_golden, 8, (2, 4), 1)


def _worker_fused_grads(rank, ws, cuda=False, transport="auto"):
    from cpu_mover import TorchCpuMover
    from paper_2509_07003_b200 import comm, create_mesh
    from paper_2509_07003_b200.dtensor import from_local
    from paper_2509_07003_b200.placement import ShardSpec, parse_placements
    if cuda:  # CUDA pack/unpack kernels, host-staged gloo collectives (see _worker_golden_cuda)
        os.environ["SDR_COMM_CPU_STAGING"] = "1"
        os.environ["SDR_TRANSPORT"] = transport
        torch.cuda.set_device(0)
        from paper_2509_07003_b200.movers import CudaMover
        mover = CudaMover()
    else:
        mover = TorchCpuMover()
    mesh = create_mesh([("dp", 2), ("tp", 2)])
    coord = mesh.coords_of_rank(rank)
    specs = ["P,P", "P,S(0)", "P,P", "R,P", "S(1),R"]
    shapes = [(6, 5), (8, 3), (3,), (4, 4), (2, 6)]
    grads, fulls = [], []
    for i, (sp, shp) in enumerate(zip(specs, shapes)):
        spec = ShardSpec(mesh, parse_placements(sp))
        from paper_2509_07003_b200.placement import local_shape_and_offset
        v = local_shape_and_offset(spec, shp, coord)
        g = torch.Generator().manual_seed(100 * i + rank)
        loc = torch.randint(-4, 5, v.local_shape, generator=g).double()
        grads.append(from_local(loc.cuda() if cuda else loc, spec, shp, coord))
    # expected: sum over the Partial fibers, computed with gathered locals
    expect = []
    for gr in grads:
        t = gr.local.cpu().clone()
        pd = gr.meta.spec.partial_mesh_dims()
        if pd:
            grp, _ = comm.fiber_group(mesh, pd)
            dist.all_reduce(t, group=grp)
        expect.append(t)
    l1, l2 = comm.CollectiveLedger(), comm.CollectiveLedger()
    out_b, rep_b = comm.bucketed_grad_reduce(grads, bucket_bytes=64, ledger=l1, mover=mover)
    out_f, rep_f = comm.fused_nd_grad_reduce(grads, bucket_bytes=1 << 20, ledger=l2, mover=mover)
    for e, b, f, g in zip(expect, out_b, out_f, grads):
        assert torch.equal(e, b.local.cpu()) and torch.equal(e, f.local.cpu())
        assert b.meta.spec == f.meta.spec
        assert not b.meta.spec.partial_mesh_dims()
    assert len(rep_b["skipped"]) == 1 and len(rep_f["skipped"]) == 1
    if cuda:
        from paper_2509_07003_b200 import peer
        assert (peer.STATS["all_reduce"] > 0) == (transport == "peer")
    # N-d fusion: the P,P group takes one round instead of one per dim
    assert len(rep_f["rounds"]) < len(rep_b["rounds"])


def test_bucketed_and_fused_grad_reduce_gloo():
    _spawn(_worker_fused_grads, 4)


def _worker_switch_reduce(rank, ws, cuda=False):
    """Opt-in reduce="switch" (NCCL / NVLS order, comm.reduce_mode): float
    sums within comm.switch_sum_tolerance of the ascending-rank float64 sum,
    integer sums exact, same buckets / rounds / ledger as the exact mode."""
    from cpu_mover import TorchCpuMover
    from paper_2509_07003_b200 import comm, create_mesh
    from paper_2509_07003_b200.dtensor import from_local
    from paper_2509_07003_b200.placement import ShardSpec, local_shape_and_offset, parse_placements
    if cuda:  # exact mode on the peer transport (ranks sharing one GPU); switch mode via host-staged gloo
        os.environ["SDR_COMM_CPU_STAGING"] = "1"
        os.environ["SDR_TRANSPORT"] = "peer"
        torch.cuda.set_device(0)
        from paper_2509_07003_b200.movers import CudaMover
        mover = CudaMover()
    else:
        mover = TorchCpuMover()
    mesh = create_mesh([("dp", 2), ("tp", 2)])
    coord = mesh.coords_of_rank(rank)
    cases = [("P,P", (33, 7), torch.float32), ("P,S(0)", (9, 4), torch.float32), ("P,P", (50,), torch.bfloat16),
             ("P,P", (6, 6), torch.float64), ("P,P", (5, 3), torch.int64)]
    grads, parts = [], []
    for i, (sp, shp, dt) in enumerate(cases):
        spec = ShardSpec(mesh, parse_placements(sp))
        v = local_shape_and_offset(spec, shp, coord)
        g = torch.Generator().manual_seed(7 * i + rank)
        loc = (torch.randint(-9, 10, v.local_shape, generator=g) if dt == torch.int64
               else torch.randn(v.local_shape, generator=g) * 10 ** (i % 3)).to(dt)
        grads.append(from_local(loc.cuda() if cuda else loc, spec, shp, coord))
        # every fiber rank's local, in ascending fiber order, for the reference sum
        grp, fib = comm.fiber_group(mesh, spec.partial_mesh_dims())
        got = [torch.empty_like(loc) for _ in fib]
        dist.all_gather(got, loc, group=grp)
        parts.append(got)
    l_ex, l_sw = comm.CollectiveLedger(), comm.CollectiveLedger()
    out_e, rep_e = comm.fused_nd_grad_reduce(grads, bucket_bytes=256, ledger=l_ex, mover=mover)
    out_s, rep_s = comm.fused_nd_grad_reduce(grads, bucket_bytes=256, ledger=l_sw, mover=mover, reduce="switch")
    assert rep_s["reduce"] == "switch" and rep_e["reduce"] == "exact"
    assert rep_s["rounds"] == rep_e["rounds"]
    assert l_sw.entries == l_ex.entries
    for (sp, shp, dt), got, e, s_ in zip(cases, parts, out_e, out_s):
        acc = got[0].clone()
        for b in got[1:]:
            acc += b  # the reference's ascending loop (comm.py:91-101)
        tol = comm.switch_sum_tolerance(sum(b.double().abs() for b in got), len(got), dt)
        if cuda or not dt.is_floating_point:
            assert torch.equal(e.local.cpu(), acc)  # peer pull (or integers): bit-identical
        else:  # CPU: gloo's own order stands in for the pull
            assert bool(((e.local.double() - acc.double()).abs() <= tol).all())
        err = (s_.local.cpu().double() - acc.double()).abs()
        assert bool((err <= tol).all()), (sp, dt, float((err - tol).max()))
        assert s_.meta.spec == e.meta.spec
    try:
        comm.fused_nd_grad_reduce(grads, reduce="nvls")
        raise AssertionError("bad reduce mode accepted")
    except comm.CommError:
        pass


def test_switch_reduce_mode_tolerance_gloo():
    _spawn(_worker_switch_reduce, 4)


@pytest.mark.gpu
def test_switch_reduce_mode_vs_peer_pull_multiprocess():
    """GPU: the exact mode runs the peer pull (bit-identical to the
    reference's ascending sum); switch mode stays within its tolerance."""
    _spawn(_worker_switch_reduce, 4, True)


def _worker_many_mixed(rank, ws):
    """Mixed dtypes in one coalesced gather; uneven shards padded per rank."""
    from cpu_mover import TorchCpuMover
    from paper_2509_07003_b200 import comm, create_mesh
    from paper_2509_07003_b200.dtensor import distribute, redistribute_many
    from paper_2509_07003_b200.placement import ShardSpec, parse_placements
    mover = TorchCpuMover()
    mesh = create_mesh([("dp", ws)])
    coord = mesh.coords_of_rank(rank)
    fulls = [torch.arange(7 * 5, dtype=torch.float32).reshape(7, 5),
             torch.arange(3 * 9, dtype=torch.int64).reshape(3, 9),
             torch.arange(2 * 3 * 10).reshape(2, 3, 10).to(torch.bfloat16),
             torch.arange(1, dtype=torch.float64)]
    specs = ["S(0)", "S(1)", "S(2)", "S(0)"]
    xs = [distribute(f, ShardSpec(mesh, parse_placements(s)), coord) for f, s in zip(fulls, specs)]
    rep = ShardSpec(mesh, parse_placements("R"))
    ledger = comm.CollectiveLedger()
    ys = redistribute_many(xs, [rep] * 4, ledger, mover=mover)
    assert ledger.count("all_gather") == 1
    for y, f in zip(ys, fulls):
        assert torch.equal(y.local, f)


def test_redistribute_many_mixed_dtypes_gloo():
    _spawn(_worker_many_mixed, 3)


def _worker_golden_cuda(rank, ws, mesh_sizes, bucket_bytes=None, transport="nccl"):
    """The same golden cases with device tensors and the CUDA pack/unpack
    kernels; every process shares cuda:0 and gloo carries the (host-staged)
    collectives (SDR_COMM_CPU_STAGING=1).  bucket_bytes forces the pipelined
    multi-bucket path (pack / side-stream collective / unpack).  transport
    "peer" maps the ranks' peer heaps through CUDA IPC (same device here) and
    runs the pack / barrier / pull kernels instead of the collectives."""
    os.environ["SDR_COMM_CPU_STAGING"] = "1"
    os.environ["SDR_TRANSPORT"] = transport
    torch.cuda.set_device(0)
    from paper_2509_07003_b200 import dtensor as DT
    if bucket_bytes is not None:
        DT.PIPELINE_BUCKET_BYTES = bucket_bytes
    from paper_2509_07003_b200 import comm, create_mesh
    from paper_2509_07003_b200.dtensor import from_local, redistribute, redistribute_many
    from paper_2509_07003_b200.movers import CudaMover
    from paper_2509_07003_b200.placement import ShardSpec, parse_placements
    man, arr = _golden()
    mover = CudaMover()
    mesh = create_mesh([(f"m{j}", s) for j, s in enumerate(mesh_sizes)])
    coord = mesh.coords_of_rank(rank)
    tag = "_".join(map(str, coord))
    cases = [c for c in man["redistribute"] if tuple(c["mesh"]) == tuple(mesh_sizes)]
    xs, dsts, wants = [], [], []
    for c in cases:
        src = ShardSpec(mesh, parse_placements(c["src"]))
        dst = ShardSpec(mesh, parse_placements(c["dst"]))
        loc = torch.from_numpy(np.ascontiguousarray(arr[c["key"] + "_in_" + tag])).cuda()
        x = from_local(loc, src, tuple(c["shape"]), coord)
        y = redistribute(x, dst, comm.CollectiveLedger(), mover=mover)
        want = arr[c["key"] + "_out_" + tag]
        assert y.local.is_cuda
        assert y.local.cpu().numpy().tobytes() == np.ascontiguousarray(want).tobytes(), (c, coord)
        xs.append(x)
        dsts.append(dst)
        wants.append(want)
    led_general = comm.CollectiveLedger()
    ys = redistribute_many(xs, dsts, led_general, mover=mover)
    for y, want, c in zip(ys, wants, cases):
        assert y.local.cpu().numpy().tobytes() == np.ascontiguousarray(want).tobytes(), ("many", c)
    from paper_2509_07003_b200 import peer
    assert (peer.STATS["all_gather"] > 0) == (transport == "peer")
    # default mover: the plan cache (peer transport) builds on the first call
    # and replays on the next; same outputs and the same ledger as above
    for rep in range(3):
        led = comm.CollectiveLedger()
        ys = redistribute_many(xs, dsts, led)
        for y, want, c in zip(ys, wants, cases):
            assert y.local.cpu().numpy().tobytes() == np.ascontiguousarray(want).tobytes(), ("plan", rep, c)
            assert y.placements == dsts[cases.index(c)].placements
        assert led.entries == led_general.entries, rep
    if transport == "peer":
        assert any(p is not DT._NO_PLAN for p in DT._PLANS.values())


@pytest.mark.gpu
@pytest.mark.parametrize("mesh_sizes,bucket,transport", [
    ((4,), None, "nccl"), ((2, 4), None, "nccl"), ((4,), 64, "nccl"), ((2, 4), 1, "nccl"),
    ((4,), None, "peer"), ((2, 4), None, "peer"), ((2, 4), 1, "peer")])
def test_redistribute_golden_cuda_movers_multiprocess(mesh_sizes, bucket, transport):
    _spawn(_worker_golden_cuda, int(np.prod(mesh_sizes)), mesh_sizes, bucket, transport)


@pytest.mark.gpu
@pytest.mark.parametrize("transport", ["nccl", "peer"])
def test_bucketed_and_fused_grad_reduce_cuda_movers_multiprocess(transport):
    _spawn(_worker_fused_grads, 4, True, transport)


def _peer_rs_inputs(q, shapes, np_dtype):
    """Rank q's Partial tensors: random non-integer values with NaN / inf
    planted at rank-specific spots (exercise the x86 NaN rules)."""
    rs = np.random.default_rng(1000 + q)
    outs = []
    for i, shp in enumerate(shapes):
        a = (rs.standard_normal(shp) * (10.0 ** rs.integers(-3, 4, shp))).astype(np.float32)
        flat = a.reshape(-1)
        if flat.size > 8:
            flat[(3 * q + i) % flat.size] = np.nan if q % 2 else -np.nan
            flat[(5 * q + 2 * i + 1) % flat.size] = np.inf if q % 3 else -np.inf
            flat[(7 * q + i + 2) % flat.size] = 1e-39 * (q + 1)  # f32 / bf16 subnormal
            flat[(11 * q + i + 4) % flat.size] = -3e-6 * (q + 1)  # f16 subnormal
        outs.append(a.astype(np_dtype))
    return outs


def _worker_peer_reduce_scatter(rank, ws, dtype_name, to_replicate=False, heap_mb=None):
    """P -> S through the peer pull kernel on non-integer data: bit-exact vs
    the reference's reduction (NumPy / ml_dtypes `acc += b` in ascending rank
    order, comm.py:113-125), NaN and inf included."""
    os.environ["SDR_COMM_CPU_STAGING"] = "1"
    os.environ["SDR_TRANSPORT"] = "peer"
    if heap_mb is not None:  # small heap: the call is cut into several buckets
        os.environ["SDR_PEER_HEAP_MB"] = str(heap_mb)
    torch.cuda.set_device(0)
    import ml_dtypes
    from paper_2509_07003_b200 import comm, create_mesh
    from paper_2509_07003_b200.dtensor import from_local, redistribute_many
    from paper_2509_07003_b200.placement import ShardSpec, parse_placements
    np_dt = {"float32": np.float32, "float16": np.float16, "bfloat16": ml_dtypes.bfloat16,
             "float64": np.float64}[dtype_name]
    t_dt = getattr(torch, dtype_name)
    mesh = create_mesh([("dp", ws)])
    coord = mesh.coords_of_rank(rank)
    shapes = [(13, 37), (8, 5, 6), (3,), (ws * 64, 128), (ws * 64, 128)]
    dsts = ["R"] * 5 if to_replicate else ["S(0)", "S(1)", "S(0)", "S(0)", "S(1)"]
    ins = [_peer_rs_inputs(q, shapes, np_dt) for q in range(ws)]
    src = ShardSpec(mesh, parse_placements("P"))
    xs = [from_local(torch.from_numpy(ins[rank][i].view(np.uint8).copy()).view(t_dt).reshape(shp).cuda(),
                     src, shp, coord) for i, shp in enumerate(shapes)]
    specs = [ShardSpec(mesh, parse_placements(d)) for d in dsts]
    ledger = comm.CollectiveLedger()
    kind = "all_reduce" if to_replicate else "reduce_scatter"
    from paper_2509_07003_b200 import peer
    regrow = heap_mb is not None and heap_mb < 0.1
    if regrow:  # a tiny first call creates a small heap; the main call must regrow it
        redistribute_many([xs[2]], [specs[2]])
    before = peer.STATS[kind]
    ys = redistribute_many(xs, specs, ledger)
    pulls = peer.STATS[kind] - before
    if regrow:
        assert peer.STATS.get("regrow", 0) == 1 and pulls >= 1, peer.STATS
    else:
        assert pulls == (1 if heap_mb is None else 2), peer.STATS
    # one ledger entry per bucket for S/P->S (as the NCCL bucket pipeline),
    # one per logical all-reduce
    assert ledger.count(kind) == (1 if to_replicate else pulls)
    for i, (y, d) in enumerate(zip(ys, dsts)):
        acc = ins[0][i].copy()
        with np.errstate(all="ignore"):
            for q in range(1, ws):
                acc += ins[q][i]
        if to_replicate:
            got = y.local.cpu().contiguous().view(torch.uint8).numpy().tobytes()
            assert got == acc.view(np.uint8).tobytes(), (dtype_name, i, rank, "R")
            continue
        dim = int(d[2])
        E = shapes[i][dim]
        c = -(-E // ws)
        lo, hi = min(E, rank * c), min(E, rank * c + c)
        want = np.ascontiguousarray(np.take(acc, np.arange(lo, hi), axis=dim))
        got = y.local.cpu().contiguous().view(torch.uint8).numpy().tobytes()
        assert got == want.view(np.uint8).tobytes(), (dtype_name, i, rank)


@pytest.mark.gpu
@pytest.mark.parametrize("dtype_name", ["float32", "bfloat16", "float16", "float64"])
def test_peer_reduce_scatter_bit_exact_nonint(dtype_name):
    _spawn(_worker_peer_reduce_scatter, 3, dtype_name)


@pytest.mark.gpu
@pytest.mark.parametrize("dtype_name", ["float32", "bfloat16"])
def test_peer_all_reduce_bit_exact_nonint(dtype_name):
    """P -> R: reduce pull + second barrier + gather pull, bit-exact vs the
    reference's ascending-rank sum (comm.py:91-101)."""
    _spawn(_worker_peer_reduce_scatter, 4, dtype_name, True)


@pytest.mark.gpu
@pytest.mark.parametrize("to_replicate", [False, True])
def test_peer_heap_regrows_for_large_member(to_replicate):
    """The first call needs a larger half than SDR_PEER_HEAP_MB gives: every
    fiber rank regrows its heap (device barrier, close, host barrier, free,
    re-exchange) and the call stays on the peer transport, bit-exact."""
    _spawn(_worker_peer_reduce_scatter, 4, "float32", to_replicate, 0.05)


@pytest.mark.gpu
@pytest.mark.parametrize("to_replicate", [False, True])
def test_peer_bucketed_small_heap(to_replicate):
    """A heap too small for the whole call: whole-member buckets, one pull
    each, still bit-exact."""
    _spawn(_worker_peer_reduce_scatter, 4, "float32", to_replicate,
           0.4 if to_replicate else 0.3)



def test_redistribute_many_bucketed_uneven_golden():
    """Bucket boundaries must not depend on a rank's (uneven) shard size:
    64-byte buckets over the golden cases, whose shards are uneven."""
    _spawn(_worker_golden, 4, (4,), 64)


def _worker_traced_redistribute(rank, ws):
    """ops.redistribute forward equals dtensor.redistribute; its backward sends
    the gradient to the source placement (Partial flipped to Replicate)."""
    from paper_2509_07003_b200 import create_mesh, ops
    from paper_2509_07003_b200.dtensor import distribute, from_local, redistribute, to_global
    from paper_2509_07003_b200.placement import ShardSpec, parse_placements
    mesh = create_mesh([("dp", ws)])
    coord = mesh.coords_of_rank(rank)
    full = torch.arange(24, dtype=torch.float64).reshape(6, 4)
    src = ShardSpec(mesh, parse_placements("S(0)"))
    dst = ShardSpec(mesh, parse_placements("R"))
    x = distribute(full, src, coord)
    x.local.requires_grad_(True)
    y = ops.redistribute(x, dst)
    assert torch.equal(y.local.detach(), full)
    w = torch.arange(24, dtype=torch.float64).reshape(6, 4) + 100 * rank
    (y.local * w).sum().backward()
    # grad of a Replicate output flows back to S(0): this rank's rows of w
    # (the replicated cotangent is used as-is, as the reference does)
    r0 = x.view.local_offset[0]
    assert torch.equal(x.local.grad, w[r0:r0 + x.local.shape[0]])


def test_traced_redistribute_gloo():
    _spawn(_worker_traced_redistribute, 2)


def _worker_golden_cpu_peer(rank, ws, mesh_sizes, initial_half):
    """The golden redistribute cases through dtensor's PEER-transport host
    logic on CPU: peer.heap_for patched to a gloo-backed stand-in with the
    same contract (tests/cpu_peer.py).  A small initial half forces whole-
    member buckets and a heap sized past it; every fiber rank must issue the
    same pulls in the same order, and the results must equal the reference's
    (regrowth itself: test_peer_heap_regrows_for_large_member on the GPU)."""
    import functools
    import cpu_peer
    from paper_2509_07003_b200 import comm, create_mesh, peer
    from paper_2509_07003_b200.dtensor import from_local, redistribute_many
    from paper_2509_07003_b200.placement import ShardSpec, parse_placements
    peer.heap_for = functools.partial(cpu_peer.heap_for, initial_half=initial_half)
    man, arr = _golden()
    mesh = create_mesh([(f"m{j}", s) for j, s in enumerate(mesh_sizes)])
    coord = mesh.coords_of_rank(rank)
    tag = "_".join(map(str, coord))
    cases = [c for c in man["redistribute"] if tuple(c["mesh"]) == tuple(mesh_sizes)]
    xs, dsts, wants = [], [], []
    for c in cases:
        src = ShardSpec(mesh, parse_placements(c["src"]))
        xs.append(from_local(torch.from_numpy(np.ascontiguousarray(arr[c["key"] + "_in_" + tag])), src,
                             tuple(c["shape"]), coord))
        dsts.append(ShardSpec(mesh, parse_placements(c["dst"])))
        wants.append(arr[c["key"] + "_out_" + tag])
    ys = redistribute_many(xs, dsts, comm.CollectiveLedger())
    for y, want, c in zip(ys, wants, cases):
        assert y.local.numpy().tobytes() == np.ascontiguousarray(want).tobytes(), ("peer-cpu", c)
    assert cpu_peer.LOG, "the peer path did not run"
    logs = [None] * ws
    dist.all_gather_object(logs, (coord, cpu_peer.LOG))
    # ranks of one fiber see identical pull sequences; all ranks pull
    assert all(l for _, l in logs), logs
    if len(mesh_sizes) == 1:
        assert len({tuple(l) for _, l in logs}) == 1, logs
    if initial_half < 1024:  # the heaps were sized (or regrown) past the initial half
        assert any(h.half > initial_half for h in cpu_peer._HEAPS.values())


@pytest.mark.parametrize("mesh_sizes,initial_half", [((4,), 1 << 20), ((2, 4), 1 << 20), ((4,), 256),
                                                     ((2, 4), 256)])
def test_peer_transport_host_logic_cpu(mesh_sizes, initial_half):
    _spawn(_worker_golden_cpu_peer, int(np.prod(mesh_sizes)), mesh_sizes, initial_half)



def _worker_uneven_rounds(rank, ws):
    """Bucket boundaries come from local_nbytes_max (the largest shard over the
    mesh, reference comm.py:140-150), so every rank cuts the same buckets even
    when its own shard is smaller: (5,4) f64 under (P, S(0)) on 2x2 gives
    shards of 96 B (tp=0) and 64 B (tp=1); two grads at 128 B per bucket make
    2 buckets on EVERY rank (local bytes would give 1 on the tp=1 ranks).
    The ledger records real (unpadded) member bytes, and the N-d fused reduce
    records the flattened mesh's name (comm.py:270)."""
    from cpu_mover import TorchCpuMover
    from paper_2509_07003_b200 import comm, create_mesh
    from paper_2509_07003_b200.dtensor import from_local
    from paper_2509_07003_b200.placement import ShardSpec, local_shape_and_offset, parse_placements
    mover = TorchCpuMover()
    mesh = create_mesh([("dp", 2), ("tp", 2)])
    coord = mesh.coords_of_rank(rank)
    spec = ShardSpec(mesh, parse_placements("P,S(0)"))
    v = local_shape_and_offset(spec, (5, 4), coord)
    grads = [from_local(torch.full(v.local_shape, float(rank + 10 * i), dtype=torch.float64), spec,
                        (5, 4), coord) for i in range(2)]
    assert grads[0].local_nbytes_max() == 96
    ledger = comm.CollectiveLedger()
    out, rep = comm.bucketed_grad_reduce(grads, bucket_bytes=128, ledger=ledger, mover=mover)
    assert len(rep["rounds"]) == 2, rep["rounds"]
    dp_peer = mesh.coords_of_rank(rank)
    other = [r for r in range(ws) if mesh.coords_of_rank(r)[1] == dp_peer[1]]
    for i, o in enumerate(out):
        assert torch.equal(o.local, torch.full(v.local_shape, float(sum(other) + 20 * i), dtype=torch.float64))
    assert [e.payload_bytes for e in ledger.entries] == [v.local_shape[0] * 4 * 8] * 2
    # N-d fusion: the ledger names the flattened mesh and counts unpadded bytes
    spec2 = ShardSpec(mesh, parse_placements("P,P"))
    g2 = [from_local(torch.ones(3, dtype=torch.float32) * rank, spec2, (3,), coord),
          from_local(torch.ones(5, dtype=torch.float32), spec2, (5,), coord)]
    l2 = comm.CollectiveLedger()
    out2, rep2 = comm.fused_nd_grad_reduce(g2, bucket_bytes=1 << 20, ledger=l2, mover=mover)
    flat = mesh.flatten_dims(["dp", "tp"])
    assert [(e.mesh, e.payload_bytes, e.participants) for e in l2.entries] == [(flat.name, 32, 4)]
    assert rep2["rounds"] == [("all_reduce", flat.name, ("dp", "tp"))]
    assert torch.equal(out2[0].local, torch.full((3,), 6.0)) and torch.equal(out2[1].local, torch.full((5,), 4.0))


def test_grad_buckets_use_local_nbytes_max_uneven_gloo():
    _spawn(_worker_uneven_rounds, 4)


def _random_cases(seed, mesh_sizes, n=10):
    """Seeded random redistribute cases (identical on every rank): shapes with
    uneven and empty shards, source placements S / R / P (a tensor dim
    sharded by at most one mesh dim), destinations S / R, mixed dtypes."""
    rs = np.random.default_rng(seed)
    cases = []
    for _ in range(n):
        nd = int(rs.integers(1, 4))
        shape = tuple(int(v) for v in rs.integers(1, 23, nd))

        def placements(allow_p):
            out, used = [], set()
            for _ in mesh_sizes:
                free = [d for d in range(nd) if d not in used]
                kind = int(rs.integers(0, 3 if allow_p else 2))
                if kind == 0 and free:
                    d = int(rs.choice(free))
                    used.add(d)
                    out.append(("S", d))
                elif kind == 2:
                    out.append(("P",))
                else:
                    out.append(("R",))
            return tuple(out)
        src, dst = placements(True), placements(False)
        has_p = any(p[0] == "P" for p in src)
        dt = ["float32", "float64", "bfloat16", "int64"][int(rs.integers(0, 4))]
        cases.append((shape, src, dst, dt, int(rs.integers(0, 1 << 30)), has_p))
    return cases


def _path_valid(shape, src, dst, mesh):
    """Whether every intermediate spec of the left-to-right walk is valid."""
    from paper_2509_07003_b200.placement import PlacementError, ShardSpec, parse_placements
    cur = list(src)
    try:
        for md in range(len(src)):
            if cur[md] != dst[md]:
                cur[md] = dst[md]
                ShardSpec(mesh, parse_placements(_pl_text(cur))).validate_for_shape(shape)
    except PlacementError:
        return False
    return True


def _local_shape(shape, pl, mesh_sizes, coord):
    from oracle import rng_oracle as O
    base = tuple(("R",) if p[0] == "P" else p for p in pl)
    return tuple(len(i) for i in O.window(shape, base, mesh_sizes, coord))


def _pl_text(pl):
    return ",".join("R" if p[0] == "R" else "P" if p[0] == "P" else f"S({p[1]})" for p in pl)


def _worker_random_peer(rank, ws, mesh_sizes, seeds):
    """Random coalesced redistributes through the peer transport (ranks share
    one GPU, CUDA IPC heaps): every rank's output equals the oracle's
    (oracle/redist_oracle.py, pinned by the golden cases) bit for bit, for
    float data too -- the pulls sum in the reference's ascending order."""
    os.environ["SDR_COMM_CPU_STAGING"] = "1"
    os.environ["SDR_TRANSPORT"] = "peer"
    torch.cuda.set_device(0)
    import ml_dtypes
    from oracle import redist_oracle as RO, rng_oracle as O
    from paper_2509_07003_b200 import create_mesh, peer
    from paper_2509_07003_b200.dtensor import from_local, redistribute_many
    from paper_2509_07003_b200.placement import ShardSpec, parse_placements
    np_dt = {"float32": np.float32, "float64": np.float64, "bfloat16": ml_dtypes.bfloat16, "int64": np.int64}
    t_dt = {"float32": torch.float32, "float64": torch.float64, "bfloat16": torch.bfloat16, "int64": torch.int64}
    mesh = create_mesh([(f"m{j}", s) for j, s in enumerate(mesh_sizes)])
    me = mesh.coords_of_rank(rank)
    from paper_2509_07003_b200.placement import PlacementError
    for seed in seeds:
        xs, dsts, wants = [], [], []
        for shape, src, dst, dt, vseed, _ in _random_cases(seed, mesh_sizes):
            if not _path_valid(shape, src, dst, mesh):
                # the reference raises PlacementError at the step that would shard a
                # tensor dim twice; so does redistribute, before any data moves
                x = from_local(torch.zeros(_local_shape(shape, src, mesh_sizes, me), device="cuda"),
                               ShardSpec(mesh, parse_placements(_pl_text(src))), shape, me)
                with pytest.raises(PlacementError):
                    redistribute_many([x], [ShardSpec(mesh, parse_placements(_pl_text(dst)))])
                continue
            rs = np.random.default_rng(vseed)
            pdims = [i for i, p in enumerate(src) if p[0] == "P"]
            base = tuple(("R",) if p[0] == "P" else p for p in src)
            glob, locs = {}, {}
            for c in O.mesh_coords(mesh_sizes):
                key = tuple(c[i] for i in pdims)  # one global per Partial coordinate
                if key not in glob:
                    g = rs.standard_normal(shape) * 10.0 ** rs.integers(-2, 3, shape)
                    glob[key] = (np.rint(g * 100) if dt == "int64" else g).astype(np_dt[dt])
                idx = O.window(shape, base, mesh_sizes, c)
                locs[c] = np.ascontiguousarray(glob[key][np.ix_(*idx)])
            out, _ = RO.redistribute(locs, shape, src, mesh_sizes, dst)
            mine = locs[me]
            t = torch.from_numpy(mine.view(np.uint16)).view(torch.bfloat16) if dt == "bfloat16" \
                else torch.from_numpy(mine)
            xs.append(from_local(t.cuda(), ShardSpec(mesh, parse_placements(_pl_text(src))), shape, me))
            dsts.append(ShardSpec(mesh, parse_placements(_pl_text(dst))))
            wants.append(np.ascontiguousarray(out[me]))
        for rep in range(2):  # general path, then the cached plan (where one applies)
            ys = redistribute_many(xs, dsts)
            for y, w, d in zip(ys, wants, dsts):
                got = y.local.cpu()
                got = got.view(torch.int16).numpy() if got.dtype == torch.bfloat16 else got.numpy()
                assert got.tobytes() == w.tobytes(), (seed, rep, d, me)
                assert y.placements == d.placements
    assert peer.STATS["all_gather"] + peer.STATS["reduce_scatter"] + peer.STATS["all_reduce"] > 0


@pytest.mark.gpu
@pytest.mark.parametrize("mesh_sizes,seeds", [((2, 2), (11, 12, 13)), ((4,), (21, 22)), ((2, 4), (31,))])
def test_random_redistribute_many_peer_vs_oracle(mesh_sizes, seeds):
    _spawn(_worker_random_peer, int(np.prod(mesh_sizes)), mesh_sizes, seeds)


def test_random_cases_are_valid_specs():
    """CPU check of the generator: every random case is a valid spec pair
    (no tensor dim sharded twice, no transition into Partial)."""
    from paper_2509_07003_b200 import create_mesh
    from paper_2509_07003_b200.placement import ShardSpec, parse_placements
    for mesh_sizes, seeds in [((2, 2), (11, 12, 13)), ((4,), (21, 22)), ((2, 4), (31,))]:
        mesh = create_mesh([(f"m{j}", s) for j, s in enumerate(mesh_sizes)])
        for seed in seeds:
            cs = _random_cases(seed, mesh_sizes)
            assert any(c[5] for c in cs)  # some Partial sources
            for shape, src, dst, *_ in cs:
                ShardSpec(mesh, parse_placements(_pl_text(src))).validate_for_shape(shape)
                ShardSpec(mesh, parse_placements(_pl_text(dst))).validate_for_shape(shape)
            assert sum(_path_valid(c[0], c[1], c[2], mesh) for c in cs) >= len(cs) // 2


def _worker_graph_peer(rank, ws, interleave=True):
    """redistribute_many captured in a CUDA graph on the peer transport (ranks
    share one GPU, IPC heaps): replays with fresh inputs written into the
    captured tensors, interleaved with eager calls on the same heaps, equal the
    reference's sums (ascending rank order) bit for bit every time."""
    os.environ["SDR_COMM_CPU_STAGING"] = "1"
    os.environ["SDR_TRANSPORT"] = "peer"
    torch.cuda.set_device(0)
    from paper_2509_07003_b200 import create_mesh, peer
    from paper_2509_07003_b200.dtensor import from_local, redistribute_many
    from paper_2509_07003_b200.placement import ShardSpec, local_shape_and_offset, parse_placements
    mesh = create_mesh([("dp", ws)])
    me = mesh.coords_of_rank(rank)
    spec = lambda t: ShardSpec(mesh, parse_placements(t))  # noqa: E731
    shapes = {"a": ((37, 5), "S(0)", "R"), "b": ((9, 13), "P", "S(0)"), "c": ((6, 7), "P", "R"),
              "d": ((4, 50), "S(1)", "R")}

    def data(step):
        """Every rank's locals for `step` (all ranks can compute all of them)."""
        out = {}
        for name, (shape, src, _) in shapes.items():
            g = torch.Generator().manual_seed(1000 * step + ord(name))  # (str hash is per-process)
            if src == "P":
                out[name] = [torch.randn(shape, generator=g) for _ in range(ws)]
            else:
                out[name] = torch.randn(shape, generator=g)
        return out

    def local(d, name, q):
        shape, src, _ = shapes[name]
        if src == "P":
            return d[name][q]
        v = local_shape_and_offset(spec(src), shape, (q,))
        sl = tuple(slice(o, o + n) for o, n in zip(v.local_offset, v.local_shape))
        return d[name][sl].contiguous()

    def expected(d, name):
        shape, src, dst = shapes[name]
        if src != "P":
            return d[name]
        acc = d[name][0].clone()
        for t in d[name][1:]:
            acc += t  # the reference's ascending loop (comm.py:91-101)
        if dst == "R":
            return acc
        v = local_shape_and_offset(spec(dst), shape, me)
        return acc[v.local_offset[0]:v.local_offset[0] + v.local_shape[0]]

    names = list(shapes)
    d0 = data(0)
    xs = [from_local(local(d0, n, rank).cuda(), spec(shapes[n][1]), shapes[n][0], me) for n in names]
    dsts = [spec(shapes[n][2]) for n in names]
    for _ in range(2):  # eager warm-up: creates (and self-checks) the heaps
        redistribute_many(xs, dsts)
    torch.cuda.synchronize()
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        redistribute_many(xs, dsts)
    torch.cuda.current_stream().wait_stream(side)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    cap0 = dict(peer.STATS)
    with torch.cuda.graph(g):
        ys = redistribute_many(xs, dsts)
    before = dict(peer.STATS)
    assert before["all_gather"] > cap0["all_gather"], (cap0, before)  # captured on the peer transport
    for step in range(1, 5):
        d = data(step)
        for x, n in zip(xs, names):
            x.local.copy_(local(d, n, rank))
        g.replay()
        # an eager call on the same heaps between replays (other data)
        e = data(100 + step)
        xe = [from_local(local(e, n, rank).cuda(), spec(shapes[n][1]), shapes[n][0], me) for n in names]
        ye = redistribute_many(xe, dsts) if interleave else []
        torch.cuda.synchronize()
        for y, n in zip(ys, names):
            got = y.local.cpu()
            if not torch.equal(got, expected(d, n)):
                stale = torch.equal(got, expected(d0, n))
                raise AssertionError((step, n, "replay", "stale" if stale else "wrong",
                                      float((got - expected(d, n)).abs().max()), rank))
        for y, n in zip(ye, names):
            assert torch.equal(y.local.cpu(), expected(e, n)), (step, n, "eager")
    # the eager calls after the capture ran on the peer transport, not NCCL
    assert peer.STATS["all_gather"] > before["all_gather"] or not interleave
    assert all(hp.captured for hp in peer._HEAPS.values() if hp.ok)


@pytest.mark.gpu
@pytest.mark.parametrize("interleave", [False, True])
def test_redistribute_many_captured_in_cuda_graph_peer(interleave):
    os.environ["SDR_PEER_TIMEOUT_S"] = "60"
    try:
        _spawn(_worker_graph_peer, 4, interleave)
    finally:
        os.environ.pop("SDR_PEER_TIMEOUT_S", None)
