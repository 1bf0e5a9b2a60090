"""Generate golden fixtures by running the REAL reference (spmdsim) here.

Run in the build container (where /root/reference exists):
    python tests/golden/make_golden.py
Writes tests/golden/*.npz + manifest.json.  The GPU box has no /root/reference;
the tests there compare against these committed fixtures and against the
oracle (oracle/), which tests/test_oracle.py pins to the same fixtures.

Cases follow the reference's own tests: test_rng.py:24-140 (golden block,
distributions x placements, theta invariance, empty shards) and
test_dtensor.py / test_comm.py (redistribute transitions).
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)

import ml_dtypes  # noqa: E402

from spmdsim import rng as R  # noqa: E402
from spmdsim.dtensor import distribute, redistribute  # noqa: E402
from spmdsim.engine import k_dropout_apply  # noqa: E402
from spmdsim.mesh import create_mesh  # noqa: E402
from spmdsim.placement import ShardSpec, local_shape_and_offset, parse_placements  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
BF16 = ml_dtypes.bfloat16


def enc(a: np.ndarray) -> tuple[np.ndarray, str]:
    """Store bf16 as its uint16 bit pattern; everything else as is."""
    a = np.asarray(a)
    if a.dtype == BF16:
        return a.view(np.uint16), "bfloat16"
    return a, a.dtype.name


def dist_of(spec):
    kind, params = spec
    return {
        "uniform01": lambda: R.Uniform01(),
        "uniform": lambda: R.Uniform(*params),
        "normal": lambda: R.Normal(*params),
        "randint": lambda: R.RandInt(*params),
        "bernoulli": lambda: R.Bernoulli(*params),
    }[kind]()


def dt_of(name):
    return BF16 if name == "bfloat16" else np.dtype(name)


def numpy_fingerprint() -> list[str]:
    u = (np.arange(0, 1 << 24, 4099, dtype=np.uint32) >> 0).astype(np.float64) * 2.0 ** -24
    r = np.sqrt(-2.0 * np.log1p(-u))
    c = np.cos(2.0 * np.pi * u)
    h = np.bitwise_xor.reduce(r.view(np.uint64)) ^ np.bitwise_xor.reduce(c.view(np.uint64) * np.uint64(3))
    return [np.__version__, hex(int(h))]


def main():
    manifest = {"numpy": numpy_fingerprint(), "philox": {}, "fills": [], "dropout": [],
                "redistribute": []}
    arrays: dict[str, np.ndarray] = {}

    # 1. Philox known answers (test_rng.py:24-46 + Random123 KATs + random triples).
    kat = [(0, 0, 0)]
    rs = np.random.default_rng(7)
    for _ in range(61):
        kat.append((int(rs.integers(0, 2 ** 63)) * 2 + int(rs.integers(0, 2)),
                    int(rs.integers(0, 2 ** 40)), int(rs.integers(0, 2 ** 62))))
    kat += [(0x12345678DEADBEEF, 123456, 2 ** 33), (2 ** 64 - 1, 2 ** 64 - 1, 2 ** 64 - 1)]
    words = [R.backend_block(s, t, b) for s, t, b in kat]
    manifest["philox"] = {"triples": [[hex(s), hex(t), hex(b)] for s, t, b in kat],
                          "words": [[hex(w) for w in ws] for ws in words]}

    # 2. Fills: distributions x dtypes x (shape, placements, mesh) x state.
    dists = [("uniform01", ()), ("uniform", (-2, 3)), ("uniform", (-0.0346, 0.0346)),
             ("normal", (0.0, 1.0)), ("normal", (0.0, 0.02)), ("normal", (2.0, 0.5)),
             ("randint", (0, 1 << 31)), ("randint", (-5, 11)),
             ("bernoulli", (0.25,)), ("bernoulli", (0.9,))]
    dtypes = {"uniform01": ["float64", "float32"],
              "uniform": ["float64", "float32", "bfloat16", "float16"],
              "normal": ["float64", "float32", "bfloat16", "float16"],
              "randint": ["float64", "int64", "int32", "float32"],
              "bernoulli": ["float64", "float32", "bfloat16", "uint8"]}
    layouts = [((16, 24), "S(0)", (4,)), ((16, 24), "S(1)", (4,)), ((16, 24), "IS(0,2)", (4,)),
               ((7, 5, 3), "S(0),S(2)", (2, 2)), ((50, 12), "S(0),S(1)", (2, 4)),
               ((33,), "S(0)", (8,)), ((2, 8), "S(0)", (4,)), ((6, 40), "R,S(1)", (2, 4))]
    states = [(7, 3, 65536), (20240817, 0, 64), (1234, 5, 7), (99, 2 ** 40, 1)]
    case = 0
    for di, d in enumerate(dists):
        for dt in dtypes[d[0]]:
            for li, (shape, pl, msizes) in enumerate(layouts):
                seed, off, th = states[(di + li) % len(states)]
                if li % 3 != case % 3 and not (li == 0):
                    case += 1
                    continue
                st = R.RngState(seed, off, th)
                ref = R.generate_global(shape, st, dist_of(d), dt_of(dt))
                mesh = create_mesh([(f"m{i}", s) for i, s in enumerate(msizes)])
                spec = ShardSpec(mesh, parse_placements(pl))
                st2 = R.RngState(seed, off, th)
                locs = R.generate_distributed(spec, shape, st2, dist_of(d), dt_of(dt))
                assert st.offset == st2.offset
                key = f"fill{case}"
                a, dname = enc(ref)
                arrays[key + "_global"] = a
                for coord, arr in locs.items():
                    arrays[key + "_local_" + "_".join(map(str, coord))] = enc(arr)[0]
                manifest["fills"].append({
                    "key": key, "dist": d[0], "params": list(d[1]), "dtype": dt, "out_dtype": dname,
                    "shape": list(shape), "placements": pl, "mesh": list(msizes),
                    "seed": seed, "offset": off, "theta": th, "offset_after": st.offset})
                case += 1

    # 3. Dropout: mask + apply, per dtype (engine.py:80-81, rng.py:238-242).
    rs = np.random.default_rng(0)
    for i, (dt, shape, p, pl, msizes) in enumerate([
            ("float32", (8, 16, 32), 0.1, "S(1)", (4,)), ("bfloat16", (8, 16, 32), 0.1, "S(1)", (2,)),
            ("float16", (4, 64), 0.3, "S(0)", (2,)), ("float64", (4, 64), 0.5, "S(1)", (4,)),
            ("bfloat16", (3, 5, 24), 0.77, "S(1)", (4,))]):
        x = rs.standard_normal(shape).astype(dt_of(dt))
        x.reshape(-1)[:4] = [0.0, -0.0, np.inf, -np.inf] if dt != "bfloat16" else x.reshape(-1)[:4]
        seed, off, th = 4242 + i, 11 * i, 65536
        mesh = create_mesh([("d", msizes[0])])
        spec = ShardSpec(mesh, parse_placements(pl))
        key = f"drop{i}"
        arrays[key + "_x"] = enc(x)[0]
        st = R.RngState(seed, off, th)
        from spmdsim.placement import full_view
        mask = R.dropout_mask_local(full_view(shape), st, p, dtype=dt_of(dt))
        y = k_dropout_apply(x, mask, p)
        arrays[key + "_mask"] = enc(mask)[0]
        arrays[key + "_y"] = enc(y)[0]
        for coord in mesh.iter_coords():
            v = local_shape_and_offset(spec, shape, coord)
            m = R.dropout_mask_local(v, st, p, dtype=dt_of(dt))
            arrays[key + "_mask_" + "_".join(map(str, coord))] = enc(m)[0]
        manifest["dropout"].append({"key": key, "dtype": dt, "shape": list(shape), "p": p,
                                    "placements": pl, "mesh": list(msizes), "seed": seed,
                                    "offset": off, "theta": th, "y_dtype": enc(y)[1]})

    # 4. Redistribute transitions on integer-valued data (test_dtensor.py style).
    rs = np.random.default_rng(3)
    cases = [((8, 6), (4,), "S(0)", "R"), ((8, 6), (4,), "S(1)", "R"), ((9, 6), (4,), "S(0)", "R"),
             ((8, 6), (4,), "P", "S(0)"), ((10, 6), (4,), "P", "S(0)"), ((8, 6), (2,), "P", "R"),
             ((8, 6), (4,), "R", "S(1)"), ((8, 6), (2,), "S(0)", "S(1)"),
             ((8, 12), (2, 4), "S(1),S(0)", "R,S(0)"), ((8, 12), (2, 4), "P,S(1)", "S(0),S(1)"),
             ((8, 12), (2, 4), "S(0),R", "R,R"), ((16, 12), (2, 4), "IS(0,2),R", "R,R")]
    for i, (shape, msizes, src, dst) in enumerate(cases):
        g = rs.integers(-4, 5, size=shape).astype(np.float64)
        mesh = create_mesh([(f"m{j}", s) for j, s in enumerate(msizes)])
        sspec = ShardSpec(mesh, parse_placements(src))
        dspec = ShardSpec(mesh, parse_placements(dst))
        x = distribute(g, sspec)
        # non-canonical Partial decomposition: random integer split
        if "P" in src:
            pdims = sspec.partial_mesh_dims()
            for coord in list(x.locals):
                if any(coord[d] != 0 for d in pdims):
                    x.locals[coord] = rs.integers(-3, 4, size=x.locals[coord].shape).astype(np.float64)
            first = {c: v for c, v in x.locals.items() if all(c[d] == 0 for d in pdims)}
            for c in first:
                others = [v for cc, v in x.locals.items() if cc != c and all(
                    cc[k] == c[k] for k in range(len(c)) if k not in pdims)]
                x.locals[c] = x.locals[c] - sum(others) if others else x.locals[c]
        key = f"redist{i}"
        for coord, arr in x.locals.items():
            arrays[key + "_in_" + "_".join(map(str, coord))] = arr
        y = redistribute(x, dspec)
        for coord, arr in y.locals.items():
            arrays[key + "_out_" + "_".join(map(str, coord))] = arr
        arrays[key + "_global"] = g
        manifest["redistribute"].append({"key": key, "shape": list(shape), "mesh": list(msizes),
                                         "src": src, "dst": dst})

    np.savez_compressed(os.path.join(OUT, "golden.npz"), **arrays)
    with open(os.path.join(OUT, "manifest.json"), "w") as f:
        json.dump(manifest, f, indent=1)
    print(f"wrote {len(arrays)} arrays, {len(manifest['fills'])} fill cases, "
          f"{len(manifest['dropout'])} dropout cases, {len(manifest['redistribute'])} redistribute cases")


if __name__ == "__main__":
    main()
