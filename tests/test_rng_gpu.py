"""GPU parity: the sm_100a RNG path vs the oracle and the reference's golden vectors.

Bit-exact for every distribution, dtype, placement, mesh and state
(reference tests test_rng.py, test_acceptance.py ac01/ac02).
"""

import math
import os

import numpy as np
import pytest
import torch

from conftest import bits, decode, numpy_fingerprint
from oracle import rng_oracle as O

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    import paper_2509_07003_b200 as S
    from paper_2509_07003_b200 import rng as R
    from paper_2509_07003_b200.placement import ShardSpec, full_view, local_shape_and_offset, parse_placements


def _dist(kind, params):
    return {"uniform01": lambda: R.Uniform01(), "uniform": lambda: R.Uniform(*params),
            "normal": lambda: R.Normal(*params), "randint": lambda: R.RandInt(*params),
            "bernoulli": lambda: R.Bernoulli(*params)}[kind]()


def _np_dt(name):
    if name == "bfloat16":
        import ml_dtypes
        return ml_dtypes.bfloat16
    return np.dtype(name)


def _oracle_tensor(a: np.ndarray) -> torch.Tensor:
    if a.dtype.name == "bfloat16":
        return torch.from_numpy(a.view(np.uint16).view(np.int16).copy()).view(torch.bfloat16)
    return torch.from_numpy(np.ascontiguousarray(a))


def _same(gpu: torch.Tensor, ref: torch.Tensor) -> bool:
    g = gpu.detach().cpu()
    return tuple(g.shape) == tuple(ref.shape) and torch.equal(bits(g), bits(ref))


def _oracle_pl(spec):
    out = []
    for p in spec.placements:
        if isinstance(p, S.Shard):
            out.append(("S", p.dim))
        elif isinstance(p, S.InterleavedShard):
            out.append(("IS", p.dim, p.interleaved_size))
        elif isinstance(p, S.Partial):
            out.append(("P",))
        else:
            out.append(("R",))
    return tuple(out)


def test_device_philox_known_answers(golden):
    man, _ = golden
    assert R.backend_block(0, 0, 0) == (0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8)
    trip = [tuple(int(v, 16) for v in t) for t in man["philox"]["triples"]]
    want = [tuple(int(v, 16) for v in w) for w in man["philox"]["words"]]
    for seed in {t[0] for t in trip}:
        sel = [i for i, t in enumerate(trip) if t[0] == seed]
        w = R.philox_blocks(seed, [trip[i][1] for i in sel], [trip[i][2] for i in sel]).cpu()
        for row, i in zip(w.tolist(), sel):
            assert tuple(row) == want[i]
    # vectorised API: beta = 2^33 carries into counter word 1 (test_rng.py:40-46)
    taus = np.array([0, 1, 65535, 123456], dtype=np.uint64)
    betas = np.array([0, 5, 7, 2 ** 33], dtype=np.uint64)
    c = [(betas & 0xFFFFFFFF).astype(np.uint32), (betas >> np.uint64(32)).astype(np.uint32),
         (taus & 0xFFFFFFFF).astype(np.uint32), (taus >> np.uint64(32)).astype(np.uint32)]
    w = R.philox_4x32_10(0xDEADBEEF, 0x12345678, *c)
    for i in range(4):
        assert tuple(int(w[j][i]) for j in range(4)) == O.block_scalar(0x12345678DEADBEEF, int(taus[i]),
                                                                       int(betas[i]))


def test_golden_fills_bit_exact(golden):
    man, arr = golden
    same_numpy = man["numpy"] == numpy_fingerprint()
    n = 0
    for c in man["fills"]:
        if c["dist"] == "normal" and not same_numpy:
            continue
        shape = tuple(c["shape"])
        dist = _dist(c["dist"], tuple(c["params"]))
        dt = _np_dt(c["dtype"])
        st = R.RngState(c["seed"], c["offset"], c["theta"])
        g = R.generate_global(shape, st, dist, dt)
        assert st.offset == c["offset_after"]
        assert _same(g, decode(arr[c["key"] + "_global"], c["out_dtype"])), c
        mesh = S.create_mesh([(f"m{i}", s) for i, s in enumerate(c["mesh"])])
        spec = ShardSpec(mesh, parse_placements(c["placements"]))
        st2 = R.RngState(c["seed"], c["offset"], c["theta"])
        locs = R.generate_distributed(spec, shape, st2, dist, dt)
        assert st2.offset == c["offset_after"]
        for coord, t in locs.items():
            ref = decode(arr[c["key"] + "_local_" + "_".join(map(str, coord))], c["out_dtype"])
            assert _same(t, ref.reshape(tuple(t.shape))), (c, coord)
        n += 1
    assert n >= 90


CASES = [
    ("uniform01", (), "float32"), ("uniform01", (), "float64"), ("uniform", (-0.5, 1.5), "float32"),
    ("uniform", (-0.0346, 0.0346), "bfloat16"), ("uniform", (-3, 7), "float64"),
    ("uniform", (-1.0, 1.0), "float16"), ("normal", (0.0, 1.0), "float32"),
    ("normal", (0.0, 0.02), "bfloat16"), ("normal", (1.5, 3.0), "float64"),
    ("normal", (-2.0, 0.5), "float16"), ("randint", (0, 1 << 31), "int64"),
    ("randint", (-7, 1000003), "float64"), ("randint", (3, 10), "int32"),
    ("bernoulli", (0.9,), "uint8"), ("bernoulli", (0.1,), "bfloat16"), ("bernoulli", (0.5,), "float32"),
]
LAYOUTS = [
    ((257, 123), "S(0)", (4,)), ((64, 96), "S(1)", (8,)), ((3, 50, 40), "S(1),S(2)", (2, 4)),
    ((48, 40), "IS(0,3),S(1)", (2, 4)), ((5, 7, 9, 11), "S(3)", (3,)), ((4097,), "S(0)", (8,)),
    ((6, 16), "R,S(0)", (2, 8)),
]


@pytest.mark.parametrize("kind,params,dt", CASES)
@pytest.mark.parametrize("theta", [65536, 64, 7, 1])
def test_sharded_fill_matches_oracle(kind, params, dt, theta):
    seed, off = 0x5EED + theta, (theta * 977) % 1000003
    for li, (shape, pl, msizes) in enumerate(LAYOUTS):
        if (li + theta) % 2 and theta != 65536:
            continue
        mesh = S.create_mesh([(f"m{i}", s) for i, s in enumerate(msizes)])
        spec = ShardSpec(mesh, parse_placements(pl))
        dist = _dist(kind, params)
        st = R.RngState(seed, off, theta)
        locs = R.generate_distributed(spec, shape, st, dist, _np_dt(dt))
        assert st.offset == O.offset_after(off, math.prod(shape), theta)
        ref = O.fill_sharded(shape, _oracle_pl(spec), msizes, seed, off, theta, kind, params, _np_dt(dt))
        for coord, t in locs.items():
            assert _same(t, _oracle_tensor(ref[coord])), (kind, dt, shape, pl, coord)
        # and bit-exact against its own unsharded 1-GPU result
        g = R.generate_global(shape, R.RngState(seed, off, theta), dist, _np_dt(dt))
        flat = g.reshape(-1)
        for coord, t in locs.items():
            v = local_shape_and_offset(spec, shape, coord)
            idx = v.global_flat_indices(device=g.device)
            assert torch.equal(bits(flat[idx]), bits(t.reshape(-1)))


def test_empty_shards_and_offsets():
    mesh = S.create_mesh([("d", 4)])
    spec = ShardSpec(mesh, parse_placements("S(0)"))
    st = R.RngState(0)
    locs = R.generate_distributed(spec, (2, 8), st, R.Uniform01())
    assert locs[(2,)].numel() == 0 and locs[(3,)].numel() == 0
    assert st.offset == 1
    st = R.RngState(0, 0, global_threads=64)
    R.generate_global((10, 10), st, R.Uniform01())
    assert st.offset == 2
    R.generate_global((4,), st, R.Uniform01())
    assert st.offset == 3


def test_beta_and_tau_carry_paths():
    """64-bit beta carries into counter word 1; tau crosses 2^32 (THETA > 2^32);
    chunks straddling a THETA boundary take the per-element path."""
    for seed, off, theta in [(1, 2 ** 32 - 3, 65536), (9, 2 ** 64 - 2, 5), (3, 0, 2 ** 32 + 5),
                             (4, 17, 12)]:
        shape = (3, 1000)
        g = R.generate_global(shape, R.RngState(seed, off, theta), R.Uniform01(), np.float64)
        j0 = 0 if theta < 2 ** 32 else 2 ** 32 - 1500  # exercise tau_lo wrap with a window
        if theta > 2 ** 32:
            # window of a huge 1-d tensor around the 32-bit tau boundary
            n = 2 ** 32 + 4000
            view = S.ShardView((n,), windows=[S.placement.DimWindow(j0, 3000)])
            t = R.fill_random(view, R.RngState(seed, off, theta), R.Uniform01(), np.float64)
            ref = O.fill_indices(np.arange(j0, j0 + 3000), seed, off, theta, "uniform01", (), np.float64)
            assert _same(t, torch.from_numpy(ref))
        ref = O.fill_global(shape, seed, off, theta, "uniform01", (), np.float64)
        assert _same(g, torch.from_numpy(ref))


def test_theta_local_thread_count_is_ignored():
    ref = R.fill_random(full_view((256,)), R.RngState(123), R.Normal(0, 1), theta=1)
    for th in (32, 1024, 65536):
        out = R.fill_random(full_view((256,)), R.RngState(123), R.Normal(0, 1), theta=th)
        assert torch.equal(bits(out), bits(ref))
    with pytest.raises(ValueError):
        R.fill_random(full_view((4,)), R.RngState(1), R.Uniform01(), theta=0)


def test_value_contracts_and_errors():
    u = R.generate_global((4096,), R.RngState(4), R.Uniform01(), dtype=np.float32)
    assert u.dtype == torch.float32
    assert bool(((u * (1 << 24)) == torch.round(u * (1 << 24))).all())
    assert R.generate_global((8,), R.RngState(4), R.Uniform01(), dtype="bfloat16").dtype == torch.float64
    r = R.generate_global((4096,), R.RngState(1), R.RandInt(5, 11))
    assert bool(((r >= 5) & (r < 11)).all())
    with pytest.raises(ValueError):
        R.Uniform(2, 1)
    with pytest.raises(ValueError):
        R.Normal(0, 0)
    with pytest.raises(ValueError):
        R.Bernoulli(1.5)
    with pytest.raises(ValueError):
        R.dropout_mask_local(full_view((4,)), R.RngState(), 1.0)
    # Uniform01 returns float64 for every non-float32 dtype (rng.py:124-127) ...
    assert R.generate_global((4,), R.RngState(), R.Uniform01(), dtype=np.int64).dtype == torch.float64
    # ... while Normal has no integer output kernel
    with pytest.raises(TypeError):
        R.generate_global((4,), R.RngState(), R.Normal(0, 1), dtype=np.int64)

    class Custom(R.Distribution):
        pass
    with pytest.raises(TypeError):
        R.generate_global((4,), R.RngState(), Custom())


def test_cfg1_randn_4096_squared_two_ranks():
    """BASELINE config 1: randn f32 [4096,4096] Shard(0) on a 2-mesh vs the
    unsharded tensor and vs the oracle (full size)."""
    shape = (4096, 4096)
    mesh = S.create_mesh([("dp", 2)])
    spec = ShardSpec(mesh, parse_placements("S(0)"))
    locs = R.generate_distributed(spec, shape, R.RngState(20240817), R.Normal(0, 1), np.float32)
    g = R.generate_global(shape, R.RngState(20240817), R.Normal(0, 1), np.float32)
    assert torch.equal(bits(torch.cat([locs[(0,)], locs[(1,)]])), bits(g))
    ref = O.fill_global(shape, 20240817, 0, 65536, "normal", (0.0, 1.0), np.float32)
    assert _same(g, torch.from_numpy(ref))


def test_cfg3_embedding_2d_mesh_uneven():
    """BASELINE config 3: [50257,4096] on dp=2 x tp=4, S(0),S(1) (25129/25128 rows),
    normal(0,0.02) and std-matched uniform, f32 and bf16: shards == 1-GPU tensor,
    and oracle spot checks across the uneven boundary."""
    shape = (50257, 4096)
    mesh = S.create_mesh([("dp", 2), ("tp", 4)])
    spec = ShardSpec(mesh, parse_placements("S(0),S(1)"))
    b = math.sqrt(3) * 0.02
    for dist, kind, params in [(R.Normal(0.0, 0.02), "normal", (0.0, 0.02)),
                               (R.Uniform(-b, b), "uniform", (-b, b))]:
        for dt in (np.float32, "bfloat16"):
            st = R.RngState(1234)
            g = R.generate_global(shape, st, dist, dt)
            for coord in [(0, 0), (1, 3), (1, 1)]:
                v = local_shape_and_offset(spec, shape, coord)
                t = R.fill_random(v, R.RngState(1234), dist, dt)
                r0, c0 = v.local_offset
                assert torch.equal(bits(t), bits(g[r0:r0 + t.shape[0], c0:c0 + t.shape[1]]))
            rows = np.arange(25125, 25133)
            cols = np.concatenate([np.arange(0, 8), np.arange(1020, 1030), np.arange(4090, 4096)])
            ref = O.fill_window(shape, [rows, cols], 1234, 0, 65536, kind, params, _np_dt(
                dt if isinstance(dt, str) else np.dtype(dt).name))
            got = g[torch.as_tensor(rows, device=g.device)][:, torch.as_tensor(cols, device=g.device)]
            assert _same(got, _oracle_tensor(ref))


def test_normal_mirror_calibration_and_large_parity():
    er, ec = R.ensure_normal_tables()
    assert er < 2 ** -36 and ec < 2 ** -46, (er, ec)  # ~2^-40 fast path, measured exhaustively
    before = R.normal_fallback_count()
    shape = (1 << 22,)
    for dt, mean, std in [(np.float32, 0.0, 1.0), ("bfloat16", 0.0, 0.02), (np.float16, 3.0, 2.0),
                          (np.float64, -1.0, 0.5)]:
        g = R.generate_global(shape, R.RngState(77), R.Normal(mean, std), dt)
        name = dt if isinstance(dt, str) else np.dtype(dt).name
        ref = O.fill_global(shape, 77, 0, 65536, "normal", (mean, std), _np_dt(name))
        assert _same(g, _oracle_tensor(ref)), name
    after = R.normal_fallback_count()
    assert after >= before


def test_normal_mirror_is_compact_and_verified():
    """The exact NumPy mirror is 2-bit ulp corrections of the device libm's
    log1p / cos (8 MiB) plus an exception list, verified bit for bit on all
    2^24 points of both functions at load (the load keeps the full 256 MiB
    tables only if that verification fails).  A reload replaces it without
    growing device memory."""
    R.ensure_normal_tables()
    info = R.normal_mirror_info()
    assert info["compact"], info
    assert info["device_bytes"] <= 8 * 2 ** 20 + 512 * 1024, info  # codes + exceptions + fast-path LUTs
    idx = torch.cuda.current_device()
    free0 = torch.cuda.mem_get_info()[0]
    R._TABLE_ERRORS.pop(idx, None)  # force a rebuild from the host's NumPy
    R.ensure_normal_tables()
    torch.cuda.synchronize()
    assert abs(torch.cuda.mem_get_info()[0] - free0) <= 16 * 2 ** 20
    assert R.normal_mirror_info()["compact"]
    # every element through the exact path (float64 output) vs the oracle
    shape = (1 << 20,)
    g = R.generate_global(shape, R.RngState(4242, 9), R.Normal(0.5, 3.0), np.float64)
    ref = O.fill_global(shape, 4242, 9, 65536, "normal", (0.5, 3.0), np.float64)
    assert _same(g, torch.from_numpy(ref))


def test_64bit_indexing_beyond_2p32_elements():
    """One launch over > 2^32 elements (u8 Bernoulli, 4.3 GB) and a small
    window at the end of a 2^40-element tensor: 64-bit j, beta and chunk math."""
    shape = (65539, 65537)  # 4,295,229,443 elements
    t = R.generate_global(shape, R.RngState(11, 3), R.Bernoulli(0.3), np.uint8)
    for r in (0, 32768, 65538):
        cols = np.array([0, 1, 7, 8, 65535, 65536])
        j = r * shape[1] + cols
        ref = O.fill_indices(j, 11, 3, 65536, "bernoulli", (0.3,), np.uint8)
        got = t[r, torch.as_tensor(cols, device=t.device)].cpu().numpy()
        assert got.tobytes() == ref.tobytes(), r
    del t
    torch.cuda.empty_cache()
    big = (1 << 20, 1 << 20)
    view = S.ShardView(big, windows=[S.placement.DimWindow((1 << 20) - 3, 3),
                                     S.placement.DimWindow((1 << 20) - 40, 40)])
    got = R.fill_random(view, R.RngState(5, 7), R.Normal(0.0, 1.0), np.float32)
    ref = O.fill_window(big, [np.arange((1 << 20) - 3, 1 << 20), np.arange((1 << 20) - 40, 1 << 20)], 5, 7,
                        65536, "normal", (0.0, 1.0), np.float32)
    assert _same(got, torch.from_numpy(ref))


def test_empty_and_single_element_windows():
    for shape in [(0,), (5, 0, 3), (1,), (1, 1, 1)]:
        t = R.generate_global(shape, R.RngState(1), R.Normal(0, 1), np.float32)
        assert tuple(t.shape) == shape
        ref = O.fill_global(shape, 1, 0, 65536, "normal", (0.0, 1.0), np.float32)
        assert _same(t, torch.from_numpy(ref))
    from paper_2509_07003_b200 import ops
    x = torch.zeros((0, 4), device="cuda")
    assert ops.dropout_apply(x, 0.5, R.RngState()).shape == (0, 4)


@pytest.mark.parametrize("cols", [1400, 1401])  # 1401: ragged rows (per-element stores, queued misses)
@pytest.mark.parametrize("dt,mean,std", [(np.float32, 0.0, 1.0), ("bfloat16", 0.0, 0.02), ("bfloat16", 3.0, 0.5),
                                         (np.float16, 3.0, 2.0), (np.float32, -7.5, 1e-3),
                                         (np.float64, 0.0, 1.0), (np.float64, -2.5, 0.3)])
def test_normal_fast_paths_equal_exact_path(dt, mean, std, cols, monkeypatch):
    """Every Normal element through the exact NumPy-table path (SDR_NORMAL_PATH=exact),
    through the float64 certified path only (=f64: for bfloat16 every element
    then misses the float32 path and goes through the per-warp queue, which
    overflows), and the default: bit-identical over 2^21 elements of an uneven
    2-D window.  float64 outputs: the mirror per element (exact) against the
    per-point corrections (f64 and default)."""
    shape = (1531, 2053)
    view = S.ShardView(shape, windows=[S.placement.DimWindow(3, 1500), S.placement.DimWindow(7, cols)])
    R.ensure_normal_tables()
    outs = {}
    for path in ("exact", "f64", None):
        if path is None:
            monkeypatch.delenv("SDR_NORMAL_PATH", raising=False)
        else:
            monkeypatch.setenv("SDR_NORMAL_PATH", path)
        before = R.normal_fallback_count()
        outs[path] = bits(R.fill_random(view, R.RngState(2024, 5, 4096), R.Normal(mean, std), dt))
        torch.cuda.synchronize()
        if path == "exact" and dt is not np.float64:  # (ragged rows: the float paths also count the discarded tail of a row's last chunk)
            n = R.normal_fallback_count() - before
            assert n == 1500 * cols or (cols % 8 and 1500 * cols <= n <= 1500 * (cols + 7))
    assert torch.equal(outs["exact"], outs["f64"]) and torch.equal(outs["exact"], outs[None])


def test_float64_normal_corrections_exhaustive():
    """float64 normals read NumPy's r[k] / c[k] as the fast functions plus a
    16-bit correction per table point (normal_chunk_f64).  Every one of the
    2^24 points of both functions goes through sdr_transform and must equal
    the oracle's float64 Box-Muller bit for bit; the corrections are resident
    (32 MiB with the double-double cosine c_cr, 48 MiB without) and only a
    few points escape to the mirror.  The same with c_cr switched off
    (SDR_NORMAL_COS_CR=0, a reload) on a sample."""
    R.ensure_normal_tables()
    info = R.normal_delta_info()
    print(info)
    # 8-bit r corrections, plus 8-bit cosine corrections and c_cr's 64 KiB table (or 16-bit ones for c_fast)
    assert 32 << 20 <= info["device_bytes"] <= 64 << 20, info
    assert 1 <= info["escapes_r"] <= 16 and info["escapes_c"] <= 1 << 14, info  # k = 0; cosine near its zeros
    n = 1 << 24
    rs = np.random.default_rng(20240917)
    k = np.arange(n, dtype=np.uint32)
    words = np.empty((4, n), dtype=np.uint32)
    words[0] = (k << np.uint32(8)) | rs.integers(0, 256, n, dtype=np.uint32)
    words[1] = (rs.permutation(k) << np.uint32(8)) | rs.integers(0, 256, n, dtype=np.uint32)
    words[2:] = 0
    for mean, std in [(0.0, 1.0), (0.5, 3.0)]:
        want = O.transform("normal", (mean, std), words, np.float64)
        got = R.Normal(mean, std).transform(tuple(words), np.float64)
        g = got.cpu().numpy()
        bad = np.flatnonzero(g.view(np.uint64) != want.view(np.uint64))
        assert bad.size == 0, (mean, std, bad[:8], g[bad[:4]], want[bad[:4]])
    idx = torch.cuda.current_device()
    try:
        os.environ["SDR_NORMAL_COS_CR"] = "0"
        R._TABLE_ERRORS.pop(idx, None)
        R.ensure_normal_tables()
        assert R.normal_delta_info()["device_bytes"] == 48 << 20
        sl = slice(0, n, 7)
        w = np.ascontiguousarray(words[:, sl])
        want = O.transform("normal", (0.5, 3.0), w, np.float64)
        got = R.Normal(0.5, 3.0).transform(tuple(w), np.float64).cpu().numpy()
        assert np.array_equal(got.view(np.uint64), want.view(np.uint64))
    finally:
        os.environ.pop("SDR_NORMAL_COS_CR", None)
        R._TABLE_ERRORS.pop(idx, None)
        R.ensure_normal_tables()


def test_randomized_windows_match_oracle():
    """150 seeded random (shape, placement, mesh, distribution, dtype, THETA)
    cases -- odd extents, ragged rows, empty and uneven shards, 1-3 mesh dims --
    every coordinate's shard against the oracle."""
    rs = np.random.default_rng(20241017)
    kinds = [("uniform01", (), "float32"), ("uniform", (-2.0, 3.0), "bfloat16"), ("normal", (0.5, 2.0), "float32"),
             ("normal", (0.0, 0.02), "bfloat16"), ("bernoulli", (0.3,), "uint8"), ("randint", (-5, 17), "int64"),
             ("normal", (1.0, 0.1), "float16"), ("uniform", (-1.0, 1.0), "float64")]
    for case in range(150):
        nd = int(rs.integers(1, 4))
        shape = tuple(int(rs.integers(1, 70 if nd > 1 else 3000)) for _ in range(nd))
        mdims = int(rs.integers(1, 3))
        msizes = tuple(int(rs.integers(1, 5)) for _ in range(mdims))
        used, pls = set(), []
        for _ in range(mdims):
            d = int(rs.integers(0, nd))
            if d in used or rs.random() < 0.3:
                pls.append("R")
            else:
                used.add(d)
                pls.append(f"S({d})")
        kind, params, dt = kinds[case % len(kinds)]
        theta = [65536, 64, 7, 1][case % 4]
        mesh = S.create_mesh([(f"m{i}", s) for i, s in enumerate(msizes)])
        spec = ShardSpec(mesh, parse_placements(",".join(pls)))
        seed, off = 1000 + case, int(rs.integers(0, 1 << 20))
        locs = R.generate_distributed(spec, shape, R.RngState(seed, off, theta), _dist(kind, params), _np_dt(dt))
        ref = O.fill_sharded(shape, _oracle_pl(spec), msizes, seed, off, theta, kind, params, _np_dt(dt))
        for coord, t in locs.items():
            assert _same(t, _oracle_tensor(ref[coord])), (case, shape, pls, msizes, kind, dt, theta, coord)


@pytest.mark.parametrize("kind,params,dt", CASES + [("uniform01", (), "bfloat16"),
                                                     ("bernoulli", (1.0,), "bool"),
                                                     ("bernoulli", (0.0,), "int64")])
def test_distribution_transform_plugin_matches_oracle(kind, params, dt):
    """Distribution.transform(words, dtype) -- the reference's distribution
    plug-in point (rng.py:104-182) -- on the GPU (sdr_transform) equals the
    oracle's transform of the same words bit for bit, and equals fill_random
    over the indices the words were drawn for."""
    rs = np.random.default_rng(abs(hash((kind, dt))) % (1 << 32))
    n = 1 << 17
    tau = rs.integers(0, 1 << 40, n, dtype=np.uint64)
    beta = rs.integers(0, 1 << 62, n, dtype=np.uint64)
    words = O.blocks(0xC0FFEE, tau, beta)  # (4, n) uint32
    want = O.transform(kind, params, words, _np_dt(dt))
    got = _dist(kind, params).transform(tuple(words), _np_dt(dt))
    assert got.is_cuda and got.shape == (n,)
    assert _same(got, _oracle_tensor(want)), (kind, params, dt)
    # torch word tensors (device, int64 holding uint32) give the same values
    tw = tuple(torch.from_numpy(w.astype(np.int64)).cuda() for w in words)
    assert _same(_dist(kind, params).transform(tw, _np_dt(dt)), _oracle_tensor(want))
    # transform(blocks of the window's counters) == fill_random of the window
    st = R.RngState(99, 12345, 64)
    shape = (37, 48)
    j = np.arange(np.prod(shape), dtype=np.uint64)
    w2 = O.blocks(99, j % np.uint64(64), j // np.uint64(64) + np.uint64(12345))
    via_words = _dist(kind, params).transform(tuple(w2), _np_dt(dt)).reshape(shape)
    via_fill = R.fill_random(full_view(shape), st, _dist(kind, params), _np_dt(dt))
    assert torch.equal(bits(via_words), bits(via_fill))


def test_distribution_transform_errors():
    words = tuple(np.zeros(4, dtype=np.uint32) for _ in range(4))
    with pytest.raises(TypeError):
        R.RandInt(0, 5).transform(words, "bfloat16")   # no bf16 randint in the reference's dtypes
    with pytest.raises(ValueError):
        R.Normal().transform(words[:2], np.float32)      # the reference unpacks 4 words

    class Custom(R.Distribution):
        pass

    with pytest.raises(TypeError):
        Custom().transform(words, np.float32)            # no kernel, no CPU fallback
    assert R.Uniform01().transform(tuple(np.zeros(0, dtype=np.uint32) for _ in range(4)),
                                   np.float32).numel() == 0


def test_allocation_tracking_is_local_sized():
    """Port of the reference's test_rng.py:124-129."""
    mesh = S.create_mesh([("x", 4)])
    spec = ShardSpec(mesh, parse_placements("S(0)"))
    with R.track_allocations() as alloc:
        R.generate_distributed(spec, (64, 64), R.RngState(0), R.Uniform01())
    assert 0 < alloc["max_elements"] <= 64 * 64 // 4


def test_normal_mirror_footprint_and_first_call_latency():
    """The exact NumPy mirror is compact (2-bit corrections, <= 9 MiB
    resident) and its first load is timed (a fresh process)."""
    import subprocess, sys, textwrap
    code = textwrap.dedent("""
        import time, torch
        torch.cuda.init(); torch.empty(1, device="cuda")
        from paper_2509_07003_b200 import rng as R
        f0 = torch.cuda.mem_get_info()[0]
        t = time.perf_counter(); R.ensure_normal_tables(); torch.cuda.synchronize()
        dt = time.perf_counter() - t
        info = R.normal_mirror_info()
        print("MIRROR", info["device_bytes"], int(info["compact"]), info["exceptions"],
              f0 - torch.cuda.mem_get_info()[0], round(dt, 3), round(info["build_ms"], 1))
    """)
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600,
                         cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    line = [l for l in out.stdout.splitlines() if l.startswith("MIRROR")]
    assert line, out.stdout + out.stderr
    nbytes, compact, nexc, delta, secs, build_ms = line[0].split()[1:]
    print(line[0])
    assert int(compact) == 1 and int(nbytes) <= 9 << 20
    # mirror + tables + the float64 corrections (64 MiB), plus the lazily loaded kernels' code
    assert int(delta) <= (24 << 20) + (64 << 20)
    assert float(secs) < 60
