"""The reference's acceptance sweep, on the GPU.

ac01 (pkg/tests/test_acceptance.py:76-106): {64K, 1M} elements x 1-5-D x
{uniform, normal, randint, dropout-mask} x P in {1,2,4,8} x every single S(d)
on a 1-D mesh and every S(d1),S(d2) pair on the 2-D factorisation
{1:(1,1), 2:(2,1), 4:(2,2), 8:(2,4)} -- merged shards must be bit-exact with
the single-device tensor, and the state must advance identically.  Here the
single-device tensor is the ORACLE's (run on this host), so every cell is also
a parity check against the reference's algorithm.

ac02 (:109-130): identical bits for local thread counts {1, 32, 1024} and for
Shard(0) vs Shard(1) on the same state.
"""

import itertools
import math

import numpy as np
import pytest
import torch

from conftest import bits
from oracle import rng_oracle as O

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    import paper_2509_07003_b200 as S
    from paper_2509_07003_b200 import rng as R
    from paper_2509_07003_b200.placement import ShardSpec, full_view, local_shape_and_offset, parse_placements

SWEEP = [("uniform01", ()), ("normal", (0.0, 1.0)), ("randint", (0, 1 << 31)), ("bernoulli", (0.5,))]
TWO_D = {1: (1, 1), 2: (2, 1), 4: (2, 2), 8: (2, 4)}


def _power_shape(numel, ndim):
    exp = int(math.log2(numel))
    base, extra = divmod(exp, ndim)
    return tuple(2 ** (base + (1 if i < extra else 0)) for i in range(ndim))


def _dist(kind, params):
    return {"uniform01": R.Uniform01, "normal": R.Normal, "randint": R.RandInt,
            "bernoulli": R.Bernoulli}[kind](*params)


@pytest.mark.parametrize("numel", [1 << 16, 1 << 20])
def test_ac01_full_sweep_bit_exact(numel):
    seed = 20240817
    checked = 0
    for ndim in range(1, 6):
        shape = _power_shape(numel, ndim)
        for kind, params in SWEEP:
            ref = torch.from_numpy(O.fill_global(shape, seed, 0, 65536, kind, params, np.float64)).cuda()
            ref_off = O.offset_after(0, numel, 65536)
            g = R.generate_global(shape, R.RngState(seed, 0), _dist(kind, params))
            assert torch.equal(bits(g), bits(ref)), (kind, shape)
            cells = []
            for P in (1, 2, 4, 8):
                m1 = S.create_mesh([("d", P)])
                cells += [(m1, f"S({d})") for d in range(ndim)]
                a, b = TWO_D[P]
                m2 = S.create_mesh([("a", a), ("b", b)])
                cells += [(m2, f"S({d1}),S({d2})") for d1, d2 in itertools.combinations(range(ndim), 2)]
            flat_ref = bits(ref).reshape(-1)
            for mesh, pl in cells:
                spec = ShardSpec(mesh, parse_placements(pl))
                st = R.RngState(seed, 0)
                locs = R.generate_distributed(spec, shape, st, _dist(kind, params))
                assert st.offset == ref_off
                merged = torch.empty_like(flat_ref)
                for coord, t in locs.items():
                    idx = local_shape_and_offset(spec, shape, coord).global_flat_indices(device="cuda")
                    merged[idx] = bits(t).reshape(-1)
                assert torch.equal(merged, flat_ref), (kind, shape, pl)
                checked += 1
    assert checked == 4 * sum(4 * (n + math.comb(n, 2)) for n in range(1, 6))


def test_ac02_theta_and_placement_invariance():
    seed = 99
    for ndim in range(1, 6):
        shape = _power_shape(1 << 16, ndim)
        for kind, params in SWEEP:
            st = R.RngState(seed, 5)
            ref = R.fill_random(full_view(shape), st, _dist(kind, params), theta=1)
            for theta in (32, 1024):
                out = R.fill_random(full_view(shape), st, _dist(kind, params), theta=theta)
                assert torch.equal(bits(out), bits(ref))
            if ndim < 2:
                continue
            mesh = S.create_mesh([("d", 4)])
            merged = {}
            for d in (0, 1):
                spec = ShardSpec(mesh, parse_placements(f"S({d})"))
                locs = R.generate_distributed(spec, shape, R.RngState(seed, 5), _dist(kind, params))
                flat = torch.empty(math.prod(shape), dtype=torch.float64, device="cuda")
                for coord, t in locs.items():
                    flat[local_shape_and_offset(spec, shape, coord).global_flat_indices(device="cuda")] = \
                        t.reshape(-1)
                merged[d] = flat.reshape(shape)
            assert torch.equal(bits(merged[0]), bits(merged[1])) and torch.equal(bits(merged[0]), bits(ref))
