"""Pin the CPU oracle (oracle/) against the reference's golden vectors.

CPU only.  The oracle is the checker of every GPU parity test, so it must
reproduce (1) the Random123 known-answer vectors and the reference's own
GOLDEN_ZERO block (pkg/tests/test_rng.py:24-30), and (2) every fixture that
tests/golden/make_golden.py produced by running the real reference.
"""

import ctypes as C
import math

import numpy as np
import pytest

from conftest import ORACLE_C, numpy_fingerprint
from oracle import redist_oracle as RO
from oracle import rng_oracle as O

GOLDEN_ZERO = (0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8)
# Random123 philox4x32-10 known-answer vectors (key 2 words, counter 4 words).
R123_KAT = [
    ((0, 0), (0, 0, 0, 0), (0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8)),
    ((0xFFFFFFFF, 0xFFFFFFFF), (0xFFFFFFFF,) * 4, (0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD)),
    ((0xA4093822, 0x299F31D0), (0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344),
     (0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1)),
]


def _pl(text):
    out = []
    for t in O_split(text):
        t = t.strip()
        if t in ("R", "P"):
            out.append((t,))
        elif t.startswith("IS("):
            d, m = t[3:-1].split(",")
            out.append(("IS", int(d), int(m)))
        else:
            out.append(("S", int(t[2:-1])))
    return tuple(out)


def O_split(text):
    items, depth, cur = [], 0, ""
    for ch in text:
        depth += (ch == "(") - (ch == ")")
        if ch == "," and depth == 0:
            items.append(cur)
            cur = ""
        else:
            cur += ch
    items.append(cur)
    return items


def _dt(name):
    if name == "bfloat16":
        import ml_dtypes
        return ml_dtypes.bfloat16
    return np.dtype(name)


def _raw(a):
    a = np.asarray(a)
    if a.dtype.name == "bfloat16":
        return a.view(np.uint16)
    return a


def test_golden_zero_and_random123_kats():
    assert O.block_scalar(0, 0, 0) == GOLDEN_ZERO
    for (k0, k1), ctr, want in R123_KAT:
        w = O.philox10(k0, k1, np.array(ctr, dtype=np.uint32).reshape(4, 1))
        assert tuple(int(x[0]) for x in w) == want


def test_philox_golden_triples(golden):
    man, _ = golden
    for (s, t, b), want in zip(man["philox"]["triples"], man["philox"]["words"]):
        got = O.block_scalar(int(s, 16), int(t, 16), int(b, 16))
        assert got == tuple(int(w, 16) for w in want)


def test_c_oracle_matches_numpy_oracle():
    lib = C.CDLL(ORACLE_C)
    out = (C.c_uint32 * 4)()
    rs = np.random.default_rng(1)
    for _ in range(200):
        s, t, b = (int(rs.integers(0, 2 ** 63)) * 2 + 1, int(rs.integers(0, 2 ** 64, dtype=np.uint64)),
                   int(rs.integers(0, 2 ** 64, dtype=np.uint64)))
        lib.oracle_block(C.c_uint64(s), C.c_uint64(t), C.c_uint64(b), out)
        assert tuple(out) == O.block_scalar(s, t, b)


def test_oracle_fills_match_reference_golden(golden):
    man, arr = golden
    same_numpy = man["numpy"] == numpy_fingerprint()
    checked = 0
    for c in man["fills"]:
        if c["dist"] == "normal" and not same_numpy:
            continue  # NumPy log1p bits differ on this host; oracle-vs-GPU tests still run
        shape = tuple(c["shape"])
        params = tuple(c["params"])
        got = O.fill_global(shape, c["seed"], c["offset"], c["theta"], c["dist"], params, _dt(c["dtype"]))
        assert _raw(got).tobytes() == arr[c["key"] + "_global"].tobytes(), c
        pls = _pl(c["placements"])
        locs = O.fill_sharded(shape, pls, c["mesh"], c["seed"], c["offset"], c["theta"], c["dist"],
                              params, _dt(c["dtype"]))
        for coord, a in locs.items():
            assert _raw(a).tobytes() == arr[c["key"] + "_local_" + "_".join(map(str, coord))].tobytes()
        assert O.offset_after(c["offset"], math.prod(shape), c["theta"]) == c["offset_after"]
        checked += 1
    assert checked >= 90


def test_oracle_dropout_matches_reference_golden(golden):
    man, arr = golden
    for c in man["dropout"]:
        dt = _dt(c["dtype"])
        x = arr[c["key"] + "_x"]
        x = x.view(dt) if c["dtype"] == "bfloat16" else x
        shape = tuple(c["shape"])
        idx = [np.arange(n) for n in shape]
        m = O.keep_mask(shape, idx, c["seed"], c["offset"], c["theta"], c["p"], dt)
        assert _raw(m).tobytes() == arr[c["key"] + "_mask"].tobytes()
        y = O.dropout_apply(x, m, c["p"])
        assert _raw(y).tobytes() == arr[c["key"] + "_y"].tobytes()


def test_c_oracle_dropout_and_uniform():
    lib = C.CDLL(ORACLE_C)
    import ml_dtypes
    rows, cols, seed, off, th = 6, 40, 77, 9, 65536
    x = np.random.default_rng(2).standard_normal((rows, cols)).astype(ml_dtypes.bfloat16)
    y = np.empty((rows, cols), np.float32)
    p = 0.1
    thr = math.ceil((1.0 - p) * 2 ** 53)
    lib.oracle_dropout_bf16(x.view(np.uint16).ctypes.data, y.ctypes.data, C.c_int64(rows), C.c_int64(cols),
                            C.c_int64(cols), C.c_int64(0), C.c_uint64(seed), C.c_uint64(off),
                            C.c_uint64(th), C.c_uint64(thr), C.c_float(np.float32(1 / (1 - p))))
    idx = [np.arange(rows), np.arange(cols)]
    m = O.keep_mask((rows, cols), idx, seed, off, th, p, ml_dtypes.bfloat16)
    assert y.tobytes() == O.dropout_apply(x, m, p).tobytes()
    u = np.empty((rows, cols), np.float32)
    lib.oracle_uniform01_f32(u.ctypes.data, C.c_int64(rows), C.c_int64(cols), C.c_int64(cols),
                             C.c_int64(0), C.c_uint64(seed), C.c_uint64(off), C.c_uint64(th))
    assert u.tobytes() == O.fill_global((rows, cols), seed, off, th, "uniform01", (), np.float32).tobytes()


def test_oracle_redistribute_matches_reference_golden(golden):
    man, arr = golden
    for c in man["redistribute"]:
        shape, msizes = tuple(c["shape"]), tuple(c["mesh"])
        locs = {}
        for coord in O.mesh_coords(msizes):
            locs[coord] = arr[c["key"] + "_in_" + "_".join(map(str, coord))]
        out, _ = RO.redistribute(locs, shape, _pl(c["src"]), msizes, _pl(c["dst"]))
        for coord, a in out.items():
            assert a.tobytes() == arr[c["key"] + "_out_" + "_".join(map(str, coord))].tobytes(), c


@pytest.mark.parametrize("n,P", [(1, 1), (5, 8), (200, 3), (64, 64), (17, 4)])
def test_oracle_sharding_never_changes_the_stream(n, P):
    ref = O.fill_global((n,), 31, 0, 65536, "uniform01", (), np.float64)
    locs = O.fill_sharded((n,), (("S", 0),), (P,), 31, 0, 65536, "uniform01", (), np.float64)
    merged = np.concatenate([locs[(k,)] for k in range(P)])
    assert merged.tobytes() == ref.tobytes()
