"""CPU tests: host-side index algebra, state, and the C-ABI library surface.

No GPU calls.  Placement / mesh semantics are checked against the oracle's
restatement of the reference (oracle/rng_oracle.py), which test_oracle.py pins
to the reference's golden fixtures.
"""

import ctypes as C
import itertools
import os
import re

import numpy as np
import pytest
from hypothesis import given, settings, strategies as st

from conftest import LIB, ROOT
from oracle import rng_oracle as O
from paper_2509_07003_b200 import _lib
from paper_2509_07003_b200.mesh import MeshError, create_mesh
from paper_2509_07003_b200.placement import (
    InterleavedShard, Partial, PlacementError, Replicate, Shard, ShardSpec, ShardView, full_view,
    local_shape_and_offset, parse_placements)
from paper_2509_07003_b200.rng import RngState


def _opl(spec):
    m = {Shard: lambda p: ("S", p.dim), Replicate: lambda p: ("R",), Partial: lambda p: ("P",),
         InterleavedShard: lambda p: ("IS", p.dim, p.interleaved_size)}
    return tuple(m[type(p)](p) for p in spec.placements)


def test_header_symbols_exported():
    hdr = open(os.path.join(ROOT, "include", "sdrng.h")).read()
    decl = set(re.findall(r"^(?:int32_t|const char\*)\s+(sdr_\w+)\(", hdr, re.M))
    assert decl == set(_lib.EXPORTED), decl ^ set(_lib.EXPORTED)
    lib = C.CDLL(LIB)
    for name in decl:
        assert hasattr(lib, name), name
    assert _lib.LIB.sdr_version() == 1
    assert _lib.LIB.sdr_strerror(_lib.E_PARAM).decode().startswith("distribution parameter")


def test_host_philox_entry_matches_oracle():
    out = (C.c_uint32 * 4)()
    for s, t, b in [(0, 0, 0), (2 ** 64 - 1, 2 ** 64 - 1, 2 ** 64 - 1), (7, 3, 9), (1, 2, 2 ** 33)]:
        assert _lib.LIB.sdr_philox_block_host(s, t, b, out) == 0
        assert tuple(out) == O.block_scalar(s, t, b)


@pytest.mark.parametrize("shape,pl,sizes", [
    ((16, 24), "S(0)", (4,)), ((16, 24), "IS(0,2)", (4,)), ((7, 5, 3), "S(0),S(2)", (2, 2)),
    ((50257, 64), "S(0),S(1)", (2, 4)), ((2, 8), "S(0)", (4,)), ((6, 40), "R,S(1)", (2, 4)),
    ((48, 40), "IS(0,3),S(1)", (2, 4)), ((9,), "P", (3,)),
])
def test_windows_match_oracle(shape, pl, sizes):
    mesh = create_mesh([(f"m{i}", s) for i, s in enumerate(sizes)])
    spec = ShardSpec(mesh, parse_placements(pl))
    for coord in mesh.iter_coords():
        v = local_shape_and_offset(spec, shape, coord)
        ref = O.window(shape, _opl(spec), sizes, coord)
        assert v.local_shape == tuple(len(i) for i in ref)
        for a, b in zip(v.index_lists, ref):
            assert np.array_equal(a, b)
        jref = O.flat_global_indices(shape, ref)
        assert np.array_equal(v.global_flat_indices(device="cpu").numpy(), jref)
        for i in range(0, v.num_local_elements, max(1, v.num_local_elements // 17)):
            assert v.local_to_global_index(i) == jref[i]
        # the C-ABI view carries the same window
        nv = v.to_native()
        assert [nv.local_len[d] for d in range(len(shape))] == list(v.local_shape)


def test_shardview_from_index_lists_roundtrip():
    v = ShardView((12, 10), [np.array([1, 2, 3, 7, 8, 9]), np.arange(10)])
    assert v.windows[0].groups == 2 and v.windows[0].group_stride == 6
    assert np.array_equal(v.index_lists[0], [1, 2, 3, 7, 8, 9])
    with pytest.raises(PlacementError):
        ShardView((12,), [np.array([0, 2, 3])])


def test_spec_validation_and_parsing():
    mesh = create_mesh([("a", 2), ("b", 2)])
    with pytest.raises(PlacementError):
        ShardSpec(mesh, parse_placements("S(0),S(0)"))
    with pytest.raises(PlacementError):
        ShardSpec(mesh, parse_placements("P,IS(0,2)"))
    with pytest.raises(PlacementError):
        ShardSpec(mesh, parse_placements("S(0)"))
    with pytest.raises(PlacementError):
        parse_placements("Q")
    s = ShardSpec(mesh, parse_placements("IS(0,2),R"))
    with pytest.raises(PlacementError):
        local_shape_and_offset(s, (6,), (0, 0))
    assert str(ShardSpec(mesh, parse_placements("S(1),P"))) == "[S(1),P]@mesh"


def test_mesh_coords_fibers_flatten():
    m = create_mesh([("dp", 2), ("tp", 4)])
    assert m.coords_of_rank(6) == (1, 2)
    assert m.rank_at((1, 3)) == 7
    assert m.submesh("dp", 2).ranks == (2, 6)
    assert m.fibers((0,)) == [[0, 4], [1, 5], [2, 6], [3, 7]]
    f = m.flatten_dims(["dp", "tp"])
    assert f.sizes == (8,) and f.ranks == tuple(range(8))
    m3 = create_mesh([("a", 2), ("b", 3), ("c", 2)])
    f3 = m3.flatten_dims(["c", "a"])
    assert f3.dims == (("a_c", 4), ("b", 3))
    assert f3.rank_at((1, 2)) == m3.rank_at((0, 2, 1))
    with pytest.raises(MeshError):
        create_mesh([("a", 2)], ranks=[0, 0])


def test_rng_state_advance():
    s = RngState(0, 0, 64)
    s.advance(100)
    assert s.offset == 2
    s.advance(0)
    assert s.offset == 2
    s.advance(65, 3)
    assert s.offset == 2 + 2 * 3
    assert s.clone() == s and s.clone() is not s
    with pytest.raises(ValueError):
        RngState(0, 0, 0)


@given(st.lists(st.integers(1, 9), min_size=1, max_size=4), st.data())
@settings(max_examples=60, deadline=None)
def test_windows_partition_the_tensor(shape, data):
    ndim = len(shape)
    P1 = data.draw(st.integers(1, 4))
    P2 = data.draw(st.integers(1, 3))
    d1 = data.draw(st.integers(0, ndim - 1))
    mesh = create_mesh([("a", P1), ("b", P2)])
    d2 = data.draw(st.integers(0, ndim - 1))
    pl = [Shard(d1), Shard(d2) if d2 != d1 else Replicate()]
    spec = ShardSpec(mesh, tuple(pl))
    seen = np.zeros(int(np.prod(shape)), dtype=np.int64)
    for coord in mesh.iter_coords():
        if d2 == d1 and coord[1] != 0:
            continue
        v = local_shape_and_offset(spec, tuple(shape), coord)
        seen[v.global_flat_indices(device="cpu").numpy()] += 1
    assert (seen == 1).all()


def test_dropout_strategy_matches_reference_dispatch():
    """Partial input -> first S(d) that validates (reduce-scatter), as the
    reference's min-byte propagation picks (dispatch.py:330-372)."""
    import torch
    from paper_2509_07003_b200.dtensor import DTensor, DTensorMeta
    from paper_2509_07003_b200.ops import dropout_input_spec
    mesh = create_mesh([("a", 2), ("b", 2)])
    for src, want in [("P,R", "S(0),R"), ("S(0),P", "S(0),S(1)"), ("S(1),S(0)", "S(1),S(0)"),
                      ("R,P", "R,S(0)"), ("P,P", "S(0),S(1)")]:
        spec = ShardSpec(mesh, parse_placements(src))
        x = DTensor(DTensorMeta((8, 8), spec, torch.float32), torch.zeros(1), (0, 0))
        assert str(dropout_input_spec(x).placements) == str(parse_placements(want)), (src, want)
        # the static-plan directive the reference records for the site (dispatch.py:619-624)
        from paper_2509_07003_b200.ops import dropout_plan_directive
        from paper_2509_07003_b200.placement import format_placements
        assert dropout_plan_directive("blk0.drop", x) == \
            f"annotate blk0.drop.<in> {format_placements(parse_placements(want))}"


@pytest.mark.parametrize("pl,sizes", [("S(0),S(1)", (2, 3)), ("P,S(1)", (2, 2)), ("IS(0,2),R", (2, 2)),
                                      ("R,R", (2, 2))])
def test_distribute_merge_roundtrip(pl, sizes):
    import torch
    from paper_2509_07003_b200.placement import distribute_local_tensors, merge_local_tensors
    mesh = create_mesh([("a", sizes[0]), ("b", sizes[1])])
    spec = ShardSpec(mesh, parse_placements(pl))
    g = torch.arange(8 * 6, dtype=torch.float64).reshape(8, 6)
    locs = distribute_local_tensors(spec, g)
    assert torch.equal(merge_local_tensors(spec, (8, 6), locs), g)
    if "R" in pl and "P" not in pl:
        bad = dict(locs)
        k = next(c for c in bad if c[1] == 1)
        bad[k] = bad[k] + 1
        with pytest.raises(PlacementError):
            merge_local_tensors(spec, (8, 6), bad)


def test_host_pipeline_blocks_tile_the_window():
    """ops._host_blocks: every local element in exactly one block, each block a
    sub-window at the right global offset."""
    import numpy as np
    from paper_2509_07003_b200 import ops
    mesh = create_mesh([("sp", 3)])
    for gshape, pl, chunks in [((18, 37, 64), "S(0)", 4), ((18, 37, 64), "S(0)", 100),
                               ((6, 111, 64), "S(1)", 32), ((8, 512, 64), "S(1)", 32), ((5,), "S(0)", 3)]:
        v = local_shape_and_offset(ShardSpec(mesh, parse_placements(pl)), gshape, (1,))
        seen = np.zeros(v.local_shape, dtype=np.int32)
        for ix, sub in ops._host_blocks(v.local_shape, v, chunks):
            seen[ix] += 1
            blk = seen[ix]
            assert blk.shape == sub.local_shape
            for d, w in enumerate(sub.windows):
                s = ix[d] if d < len(ix) else slice(None)
                start = (s.start or 0) if isinstance(s, slice) else s
                assert w.start == v.windows[d].start + start
        assert (seen == 1).all(), (gshape, pl, chunks)


def test_reference_top_level_exports_present():
    """Every name the reference package exports at top level
    (spmdsim/__init__.py:3-32) is importable from this package."""
    import paper_2509_07003_b200 as S
    ref = ["DeviceMesh", "create_mesh", "Placement", "Shard", "Replicate", "Partial", "InterleavedShard",
           "ShardSpec", "ShardView", "DTensor", "DTensorMeta", "distribute", "redistribute", "to_global",
           "RngState"]
    assert [n for n in ref if not hasattr(S, n)] == []
    assert set(ref) <= set(S.__all__)


def test_single_process_collectives_match_reference():
    """comm.all_reduce / all_gather / reduce_scatter (single-process forms)
    against the reference's on the same buffers (ascending-rank sums)."""
    import torch
    from paper_2509_07003_b200 import comm as C2
    ref = _ref_module("comm")
    g = np.random.default_rng(3)
    bufs = [g.standard_normal((5, 6)) for _ in range(4)]
    tb = [torch.from_numpy(b) for b in bufs]
    assert np.array_equal(C2.all_reduce(tb).numpy(), ref.all_reduce(bufs))
    assert [t.numpy().tobytes() for t in C2.all_gather(tb)] == [b.tobytes() for b in ref.all_gather(bufs)]
    sl = lambda a, k: a[k:k + 1]
    got = C2.reduce_scatter(tb, sl)
    want = ref.reduce_scatter(bufs, sl)
    assert all(np.array_equal(a.numpy(), b) for a, b in zip(got, want))
    b = C2.GradBucket(100)
    assert b.fits(1000) and not (b.members.append(1) or b.fits(1000))


def test_reference_module_names_present():
    """Every public function/class of the reference's rng / placement / mesh /
    dtensor / comm modules has a same-named counterpart here."""
    import importlib
    import inspect
    for mod in ["rng", "placement", "mesh", "dtensor", "comm"]:
        r = _ref_module(mod)
        o = importlib.import_module("paper_2509_07003_b200." + mod)
        names = [n for n, v in vars(r).items() if not n.startswith("_") and
                 (inspect.isfunction(v) or inspect.isclass(v)) and getattr(v, "__module__", "") == r.__name__]
        assert [n for n in names if not hasattr(o, n)] == [], mod


def test_reference_class_methods_present():
    """Public methods of the reference's core classes exist here too (DTensor's
    per-rank forms, RngState, ShardSpec / ShardView, DeviceMesh, ledger)."""
    import importlib
    pairs = [("rng", "RngState"), ("placement", "ShardSpec"), ("placement", "ShardView"),
             ("dtensor", "DTensor"), ("dtensor", "DTensorMeta"), ("mesh", "DeviceMesh")]
    for mod, cls in pairs:
        r = getattr(_ref_module(mod), cls)
        o = getattr(importlib.import_module("paper_2509_07003_b200." + mod), cls)
        assert [n for n in dir(r) if not n.startswith("_") and not hasattr(o, n)] == [], (mod, cls)


def _ref_module(name):
    import importlib
    import sys
    ref_src = "/root/reference/pkg/src"
    if not os.path.isdir(ref_src):
        pytest.skip("reference not mounted (only in the build container)")
    if ref_src not in sys.path:
        sys.path.insert(0, ref_src)
    return importlib.import_module("spmdsim." + name)


def test_peer_transport_selection(monkeypatch):
    """SDR_TRANSPORT parsing and the cases that must stay on NCCL without
    touching the GPU: no process group, CPU tensors, forced nccl."""
    import torch
    from paper_2509_07003_b200 import peer
    monkeypatch.setenv("SDR_TRANSPORT", "bogus")
    with pytest.raises(ValueError):
        peer.transport()
    for t in ("auto", "peer", "nccl"):
        monkeypatch.setenv("SDR_TRANSPORT", t)
        assert peer.transport() == t
        assert peer.heap_for(None, [0, 1], torch.device("cpu")) is None
        assert peer.heap_for(object(), [0, 1], torch.device("cpu")) is None
    monkeypatch.setenv("SDR_TRANSPORT", "nccl")
    assert peer.heap_for(object(), [0, 1], torch.device("cuda", 0)) is None
    assert peer.reducible(torch.bfloat16) and not peer.reducible(torch.bool)


def test_dropout_buffer_validation():
    """ops._check_buffer guards every caller-supplied buffer the dropout kernel
    writes through a raw pointer (wrong dtype -> TypeError; shape, device or
    layout -> ValueError), as fill_random does for `out`."""
    import torch
    from paper_2509_07003_b200.ops import _check_buffer
    x = torch.zeros(4, 6, dtype=torch.bfloat16)
    _check_buffer("out", torch.empty(4, 6, dtype=torch.bfloat16), x, (torch.bfloat16,))
    with pytest.raises(TypeError):
        _check_buffer("out", torch.empty(4, 6, dtype=torch.float16), x, (torch.bfloat16,))
    with pytest.raises(TypeError):
        _check_buffer("mask", [0] * 24, x, (torch.uint8,))
    with pytest.raises(ValueError):
        _check_buffer("out", torch.empty(4, 5, dtype=torch.bfloat16), x, (torch.bfloat16,))
    with pytest.raises(ValueError):
        _check_buffer("out", torch.empty(6, 4, dtype=torch.bfloat16).t(), x, (torch.bfloat16,))
    with pytest.raises(ValueError):
        _check_buffer("mask", torch.empty(4, 6, dtype=torch.uint8, device="meta"), x, (torch.uint8,))


def test_cost_model_matches_reference():
    """comm.cost_model_eval against the reference's pinned values
    (test_comm.py:157-175, test_acceptance.py:289-318): T_v = 2SB sum (P_i-1)/P_i,
    T_f = 2SB (prod P - 1)/prod P; 4/3 at (2,2), 1.778 at (8,8)."""
    from fractions import Fraction
    from paper_2509_07003_b200.comm import CommError, CostParams, cost_model_eval
    tv, tf, r = cost_model_eval(CostParams(1000, Fraction(1, 100), (2, 2)))
    assert (tv, tf, r) == (Fraction(20), Fraction(15), Fraction(4, 3))
    _, _, r88 = cost_model_eval(CostParams(1 << 20, Fraction(1), (8, 8)))
    assert r88 == Fraction(7 * 2 * 64, 8 * 63) and abs(float(r88) - 1.778) < 1e-3
    assert cost_model_eval(CostParams(8, Fraction(1), (4,)))[2] == 1  # one dim: nothing to fuse
    for p in [(2,), (2, 2), (2, 4), (8, 8), (2, 2, 2)]:  # fusing never costs more
        tv, tf, r = cost_model_eval(CostParams(64, Fraction(3), p))
        assert tf <= tv and r >= 1
    with pytest.raises(CommError):
        CostParams(0, Fraction(1), (2,))
    with pytest.raises(CommError):
        CostParams(8, Fraction(1), ())
    with pytest.raises(CommError):
        CostParams(8, Fraction(1), (0, 2))


def test_cost_model_ac07_and_ledger_bytes():
    """Reference acceptance ac07 (test_acceptance.py:289-318): exact rational
    formulas, ratio -> N at P_i = 2^10, ledger 2S(P-1)/P per device; plus
    test_comm.py:167-172 (fused == vanilla iff one dim)."""
    import math
    from fractions import Fraction
    from paper_2509_07003_b200.comm import CostParams, all_reduce, cost_model_eval
    from paper_2509_07003_b200.ledger import CollectiveLedger
    B = Fraction(1, 10 ** 9)
    for N in (1, 2, 3):
        for counts in itertools.product((2, 4, 8, 16), repeat=N):
            tv, tf, ratio = cost_model_eval(CostParams(4096, B, counts))
            ev = 2 * 4096 * B * sum(Fraction(p - 1, p) for p in counts)
            prod = math.prod(counts)
            ef = 2 * 4096 * B * Fraction(prod - 1, prod)
            assert (tv, tf, ratio) == (ev, ef, ev / ef)
            assert (tf == tv) == (N == 1)
        _, _, ratio = cost_model_eval(CostParams(1, B, tuple([1 << 10] * N)))
        assert abs(float(ratio) - N) / N <= 1e-3
    import torch
    for P in (2, 4, 8, 16):
        ledger = CollectiveLedger()
        all_reduce([torch.zeros(128, dtype=torch.float64) for _ in range(P)], ledger)
        assert ledger.entries[0].bytes_per_device == Fraction(2 * 1024 * (P - 1), P)


def test_redistribute_rejects_double_sharding_path_like_reference():
    """The reference raises PlacementError when a left-to-right step would
    shard a tensor dim by two mesh dims (dtensor.py:208-258), e.g.
    [S(0),S(1)] -> [S(1),S(0)]; redistribute_many checks the whole walk
    before any collective, so it raises the same error on every rank."""
    import torch
    from paper_2509_07003_b200 import create_mesh
    from paper_2509_07003_b200.dtensor import from_local, redistribute_many
    from paper_2509_07003_b200.placement import PlacementError, ShardSpec, local_shape_and_offset, parse_placements
    mesh = create_mesh([("a", 2), ("b", 2)])
    for s, d in [("S(0),S(1)", "S(1),S(0)"), ("P,S(0)", "S(0),R"), ("R,S(0)", "S(0),R")]:
        src = ShardSpec(mesh, parse_placements(s))
        v = local_shape_and_offset(src, (6, 8), (0, 0))
        x = from_local(torch.zeros(v.local_shape), src, (6, 8), (0, 0))
        with pytest.raises(PlacementError):
            redistribute_many([x], [ShardSpec(mesh, parse_placements(d))])


def test_cos_cr_constants_split_pi_over_1024():
    """c_cr's argument reduction (dist_transforms.cuh): pi/1024 = kQ1 + kQ2 +
    kQ3 to about 2^-110, with kQ1 and kQ2 of at most 40 significant bits so
    that i*kQ1 and i*kQ2 are exact for every table index i <= 2048."""
    import re
    from decimal import Decimal, getcontext
    from fractions import Fraction
    src = open(os.path.join(ROOT, "paper_2509_07003_b200", "csrc", "dist_transforms.cuh")).read()
    m = re.search(r"kQ1 = (\S+), kQ2 = (\S+), kQ3 = (\S+);", src)
    assert m, "constants not found"
    q = [float.fromhex(x) for x in m.groups()]
    getcontext().prec = 60
    pi = Fraction(Decimal("3.14159265358979323846264338327950288419716939937510582097494459"))
    err = abs(sum(Fraction(x) for x in q) - pi / 1024)
    assert err < Fraction(1, 2 ** 110), float(err)
    import math
    for x in q[:2]:
        m53 = int(math.frexp(x)[0] * 2 ** 53)  # the 53-bit significand as an integer
        assert m53 % 2 ** 13 == 0, x           # at most 40 significant bits
        assert 2048 * (m53 >> 13) < 2 ** 53     # i * q exact for i <= 2048
