"""NumPy restatement of the reference's single-device-semantic distributed RNG.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Each function cites the
reference file:line it restates; paths are relative to
/root/reference/pkg/src/spmdsim/.

Placements are plain tuples here so the oracle shares no code with the product:
    ("S", d)       Shard(d)              placement.py:36-41
    ("R",)         Replicate             placement.py:44-47
    ("P",)         Partial(sum)          placement.py:50-55
    ("IS", d, m)   InterleavedShard(d,m) placement.py:58-64
"""

from __future__ import annotations

import math

import numpy as np

U32 = np.uint32
U64 = np.uint64
MASK32 = 0xFFFFFFFF
MASK64 = 0xFFFFFFFFFFFFFFFF

# Philox4x32 multipliers and Weyl key increments (rng.py:26-29).
PHILOX_M = (0xD2511F53, 0xCD9E8D57)
PHILOX_W = (0x9E3779B9, 0xBB67AE85)


# ---------------------------------------------------------------------------
# Philox4x32-10 (rng.py:34-59)
# ---------------------------------------------------------------------------

def philox10(key_lo: int, key_hi: int, ctr: np.ndarray) -> np.ndarray:
    """Ten Philox rounds over a (4, n) uint32 counter array -> (4, n) words.

    Round r (rng.py:46-58): the two 32x32->64 products M0*x0 and M1*x2 are
    split into hi/lo halves; x <- (hi1^x1^k0, lo1, hi0^x3^k1, lo0); the key
    is bumped by the Weyl constants after every round."""
    x = np.asarray(ctr, dtype=U32).copy()
    keys = [key_lo & MASK32, key_hi & MASK32]
    m0, m1 = U64(PHILOX_M[0]), U64(PHILOX_M[1])
    for _ in range(10):
        prod_a = x[0].astype(U64) * m0
        prod_b = x[2].astype(U64) * m1
        hi_a = (prod_a >> U64(32)).astype(U32)
        hi_b = (prod_b >> U64(32)).astype(U32)
        nxt = np.empty_like(x)
        nxt[0] = hi_b ^ x[1] ^ U32(keys[0])
        nxt[1] = prod_b.astype(U32)          # low half (truncating cast)
        nxt[2] = hi_a ^ x[3] ^ U32(keys[1])
        nxt[3] = prod_a.astype(U32)
        x = nxt
        keys = [(keys[0] + PHILOX_W[0]) & MASK32, (keys[1] + PHILOX_W[1]) & MASK32]
    return x


def counter_words(tau: np.ndarray, beta: np.ndarray) -> np.ndarray:
    """Counter layout of `_blocks_for` (rng.py:76-80): lanes 0/1 = 64-bit
    virtual offset beta (lo, hi), lanes 2/3 = 64-bit virtual thread tau."""
    tau = np.asarray(tau, dtype=U64)
    beta = np.asarray(beta, dtype=U64)
    lo = U64(MASK32)
    return np.stack([
        (beta & lo).astype(U32), (beta >> U64(32)).astype(U32),
        (tau & lo).astype(U32), (tau >> U64(32)).astype(U32),
    ])


def blocks(seed: int, tau, beta) -> np.ndarray:
    """Philox words for (seed, tau, beta) arrays; seed masked to 64 bits and
    split into the two key halves (rng.py:81-82)."""
    s = int(seed) & MASK64
    return philox10(s & MASK32, s >> 32, counter_words(tau, beta))


def block_scalar(seed: int, tau: int, beta: int) -> tuple[int, int, int, int]:
    """Scalar form of `backend_block` (rng.py:62-73)."""
    w = blocks(seed, np.array([tau], dtype=U64), np.array([beta], dtype=U64))
    return tuple(int(w[i][0]) for i in range(4))


# ---------------------------------------------------------------------------
# Shared generator state (rng.py:85-101)
# ---------------------------------------------------------------------------

def ceil_div(a: int, b: int) -> int:
    return -(-a // b)


def offset_after(offset: int, global_numel: int, theta: int, k: int = 1) -> int:
    """offset += ceil(numel / THETA) * K  (rng.py:95-98)."""
    return offset + ceil_div(global_numel, theta) * k


# ---------------------------------------------------------------------------
# Index algebra (placement.py:202-257, mesh.py:66-92)
# ---------------------------------------------------------------------------

def mesh_coords(sizes):
    """Row-major coordinates of every device (mesh.py:90-92)."""
    import itertools
    return list(itertools.product(*(range(s) for s in sizes)))


def ceil_block(length: int, parts: int, k: int) -> tuple[int, int]:
    """Ceil-block split (placement.py:226-231)."""
    b = ceil_div(length, parts)
    lo = min(k * b, length)
    return lo, min(lo + b, length)


def window(global_shape, placements, mesh_sizes, coord) -> list[np.ndarray]:
    """Per-tensor-dim ascending global coordinates owned by `coord`
    (local_shape_and_offset, placement.py:234-257)."""
    idx = [np.arange(n, dtype=np.int64) for n in global_shape]
    for md, pl in enumerate(placements):
        P, k = mesh_sizes[md], coord[md]
        if pl[0] == "S":
            lo, hi = ceil_block(global_shape[pl[1]], P, k)
            idx[pl[1]] = np.arange(lo, hi, dtype=np.int64)
        elif pl[0] == "IS":
            d, m = pl[1], pl[2]
            glen = global_shape[d] // m
            per = glen // P
            idx[d] = np.concatenate([
                np.arange(g * glen + k * per, g * glen + (k + 1) * per, dtype=np.int64)
                for g in range(m)]) if m else np.zeros(0, np.int64)
    return idx


def row_major_strides(shape) -> list[int]:
    st = [1] * len(shape)
    for d in range(len(shape) - 2, -1, -1):
        st[d] = st[d + 1] * shape[d + 1]
    return st


def flat_global_indices(global_shape, idx_lists) -> np.ndarray:
    """j = sum_d idx_d * pi_d in local row-major order
    (ShardView.global_flat_indices, placement.py:213-223)."""
    local_shape = [len(ix) for ix in idx_lists]
    n = math.prod(local_shape)
    if n == 0:
        return np.zeros(0, dtype=np.int64)
    strides = row_major_strides(global_shape)
    j = np.zeros(local_shape, dtype=np.int64)
    nd = len(global_shape)
    for d in range(nd):
        shp = [1] * nd
        shp[d] = local_shape[d]
        j = j + (idx_lists[d].astype(np.int64) * strides[d]).reshape(shp)
    return j.reshape(-1)


# ---------------------------------------------------------------------------
# Distribution transforms (rng.py:113-182)
# ---------------------------------------------------------------------------

def _u24(w) -> np.ndarray:
    """24-bit uniform in [0,1) from one word, as float64 (rng.py:113-115)."""
    return (w >> U32(8)).astype(np.float64) * 2.0 ** -24


def _u64(w0, w1) -> np.ndarray:
    return w0.astype(U64) | (w1.astype(U64) << U64(32))


def _u53(w0, w1) -> np.ndarray:
    """53-bit uniform in [0,1) from words 0-1 (rng.py:126-127)."""
    return (_u64(w0, w1) >> U64(11)).astype(np.float64) * 2.0 ** -53


def transform(kind: str, params: tuple, words: np.ndarray, dtype) -> np.ndarray:
    """Map Philox words to values, replicating NumPy-2 dtype semantics.

    kind/params:
      "uniform01", ()           Uniform01 (rng.py:118-127): f32 -> 24-bit;
                                any other dtype -> float64 53-bit (NOT cast).
      "uniform", (lo, hi)       Uniform (rng.py:130-138): f32 arithmetic for
                                f32 (weak Python scalars), else f64 then cast.
      "normal", (mean, std)     Normal (rng.py:141-156): f64 Box-Muller on
                                words 0/1, then cast.
      "randint", (lo, hi)       RandInt (rng.py:159-171): lo + u64 % span.
      "bernoulli", (p,)         Bernoulli (rng.py:174-182): 53-bit u < p.
    """
    dtype = np.dtype(dtype)
    w0, w1 = words[0], words[1]
    if kind == "uniform01":
        if dtype == np.float32:
            return _u24(w0).astype(np.float32)
        return _u53(w0, w1)
    if kind == "uniform":
        lo, hi = params
        if dtype == np.float32:
            u = _u24(w0).astype(np.float32)
            return (lo + (hi - lo) * u).astype(dtype)
        u = _u53(w0, w1)
        return (lo + (hi - lo) * u).astype(dtype)
    if kind == "normal":
        mean, std = params
        u1 = _u24(w0)
        u2 = _u24(w1)
        radius = np.sqrt(-2.0 * np.log1p(-u1))
        z = radius * np.cos(2.0 * np.pi * u2)
        return (mean + std * z).astype(dtype)
    if kind == "randint":
        lo, hi = params
        span = U64(hi - lo)
        return (lo + (_u64(w0, w1) % span).astype(np.int64)).astype(dtype)
    if kind == "bernoulli":
        (p,) = params
        return (_u53(w0, w1) < p).astype(dtype)
    raise ValueError(f"unknown distribution {kind!r}")


# ---------------------------------------------------------------------------
# Fills (rng.py:185-242)
# ---------------------------------------------------------------------------

def fill_indices(j: np.ndarray, seed: int, offset: int, theta: int, kind: str,
                 params: tuple, dtype) -> np.ndarray:
    """Values for global flat indices j (fill_random, rng.py:198-203):
    tau = j mod THETA, beta = j div THETA + offset (uint64 wrap)."""
    j = np.asarray(j, dtype=np.int64).astype(U64)
    th = U64(theta)
    tau = j % th
    beta = j // th + U64(int(offset) & MASK64)
    return transform(kind, params, blocks(seed, tau, beta), dtype)


def fill_window(global_shape, idx_lists, seed, offset, theta, kind, params, dtype):
    """One device's local window, reshaped to its local shape."""
    j = flat_global_indices(global_shape, idx_lists)
    vals = fill_indices(j, seed, offset, theta, kind, params, dtype)
    return vals.reshape([len(ix) for ix in idx_lists])


def fill_global(global_shape, seed, offset, theta, kind, params, dtype):
    """generate_global without the state advance (rng.py:208-217)."""
    idx = [np.arange(n, dtype=np.int64) for n in global_shape]
    return fill_window(global_shape, idx, seed, offset, theta, kind, params, dtype)


def fill_sharded(global_shape, placements, mesh_sizes, seed, offset, theta, kind,
                 params, dtype) -> dict:
    """generate_distributed without the state advance (rng.py:220-235)."""
    out = {}
    for coord in mesh_coords(mesh_sizes):
        idx = window(global_shape, placements, mesh_sizes, coord)
        out[coord] = fill_window(global_shape, idx, seed, offset, theta, kind, params, dtype)
    return out


def keep_mask(global_shape, idx_lists, seed, offset, theta, p, dtype):
    """dropout_mask_local (rng.py:238-242): Bernoulli(1 - p), p in [0, 1)."""
    if not 0.0 <= p < 1.0:
        raise ValueError(f"dropout needs p in [0, 1), got {p}")
    return fill_window(global_shape, idx_lists, seed, offset, theta, "bernoulli",
                       (1.0 - p,), dtype)


def dropout_apply(x: np.ndarray, mask: np.ndarray, p: float) -> np.ndarray:
    """engine.k_dropout_apply (engine.py:80-81) under NumPy-2 promotion:
    (x * m) * (1/(1-p)), the Python-float scale a weak scalar."""
    return x * mask * (1.0 / (1.0 - p))


def merge(global_shape, placements, mesh_sizes, locals_: dict, dtype) -> np.ndarray:
    """Scatter every device's window back by global flat index (the merge used
    by the reference's sweep tests, test_acceptance.py:68-73)."""
    flat = np.zeros(math.prod(global_shape), dtype=dtype)
    for coord, arr in locals_.items():
        idx = window(global_shape, placements, mesh_sizes, coord)
        flat[flat_global_indices(global_shape, idx)] = np.asarray(arr).reshape(-1)
    return flat.reshape(global_shape)
