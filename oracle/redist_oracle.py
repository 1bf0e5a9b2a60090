"""NumPy restatement of the reference's placement redistribution.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Restates
/root/reference/pkg/src/spmdsim/dtensor.py:166-298 and comm.py:91-125 on a
dict {mesh_coord: ndarray} with tuple placements (see rng_oracle docstring).
Reductions run in ascending fiber-rank order like comm.all_reduce
(comm.py:97-99) / comm.reduce_scatter (comm.py:120-122).
"""

from __future__ import annotations

import numpy as np

from .rng_oracle import mesh_coords, window


def _fibers(mesh_sizes, mesh_dim):
    """Coordinate lists, one per fiber along mesh_dim (dtensor.py:185-198)."""
    seen = []
    for c in mesh_coords(mesh_sizes):
        key = c[:mesh_dim] + c[mesh_dim + 1:]
        if key in seen:
            continue
        seen.append(key)
        yield [c[:mesh_dim] + (k,) + c[mesh_dim + 1:] for k in range(mesh_sizes[mesh_dim])]


def _with(placements, md, pl):
    out = list(placements)
    out[md] = pl
    return tuple(out)


def _positions(base: np.ndarray, wanted: np.ndarray) -> np.ndarray:
    where = {int(g): i for i, g in enumerate(base)}
    return np.array([where[int(g)] for g in wanted], dtype=np.int64)


def gather_dim(locals_, global_shape, placements, mesh_sizes, md):
    """Shard/IS -> Replicate along mesh dim md: every fiber member receives the
    fiber's shards placed at their coordinates (dtensor.py:219-227, 261-283)."""
    tdim = placements[md][1]
    rep = _with(placements, md, ("R",))
    out = {}
    for fiber in _fibers(mesh_sizes, md):
        base = window(global_shape, rep, mesh_sizes, fiber[0])[tdim]
        shape = list(np.shape(locals_[fiber[0]]))
        shape[tdim] = len(base)
        buf = np.zeros(shape, dtype=locals_[fiber[0]].dtype)
        for c in fiber:
            own = window(global_shape, placements, mesh_sizes, c)
            if np.prod([len(i) for i in own]) == 0:
                continue
            sl = [slice(None)] * len(shape)
            sl[tdim] = _positions(base, own[tdim])
            buf[tuple(sl)] = locals_[c]
        for c in fiber:
            out[c] = buf.copy()
    return out, rep


def _slice_piece(buf, global_shape, placements, mesh_sizes, coord, md, dst):
    tdim = dst[1]
    base = window(global_shape, _with(placements, md, ("R",)), mesh_sizes, coord)[tdim]
    want = window(global_shape, _with(placements, md, dst), mesh_sizes, coord)[tdim]
    sl = [slice(None)] * buf.ndim
    sl[tdim] = _positions(base, want)
    return np.ascontiguousarray(buf[tuple(sl)])


def reduce_dim(locals_, global_shape, placements, mesh_sizes, md, dst):
    """Partial -> Replicate (all-reduce) or Partial -> Shard (reduce-scatter)
    along md, summing in ascending fiber order (dtensor.py:229-245)."""
    out = {}
    for fiber in _fibers(mesh_sizes, md):
        acc = locals_[fiber[0]].copy()
        for c in fiber[1:]:
            acc += locals_[c]
        for c in fiber:
            if dst[0] == "R":
                out[c] = acc.copy()
            else:
                out[c] = _slice_piece(acc, global_shape, placements, mesh_sizes, c, md, dst)
    return out, _with(placements, md, dst)


def slice_dim(locals_, global_shape, placements, mesh_sizes, md, dst):
    """Replicate -> Shard/IS: local slice, no communication (dtensor.py:247-251)."""
    out = {c: _slice_piece(locals_[c], global_shape, placements, mesh_sizes, c, md, dst)
           for c in locals_}
    return out, _with(placements, md, dst)


def redistribute(locals_, global_shape, placements, mesh_sizes, dst_placements):
    """Mesh dims left to right, skipping equal placements (dtensor.py:166-182)."""
    cur = tuple(placements)
    for md in range(len(mesh_sizes)):
        src, dst = cur[md], dst_placements[md]
        if src == dst:
            continue
        if dst[0] == "P":
            raise ValueError("transition into Partial is unsupported")
        if src[0] in ("S", "IS") and dst[0] == "R":
            locals_, cur = gather_dim(locals_, global_shape, cur, mesh_sizes, md)
        elif src[0] == "P":
            locals_, cur = reduce_dim(locals_, global_shape, cur, mesh_sizes, md, dst)
        elif src[0] == "R":
            locals_, cur = slice_dim(locals_, global_shape, cur, mesh_sizes, md, dst)
        else:  # shard -> shard: gather then slice (dtensor.py:253-256)
            locals_, cur = gather_dim(locals_, global_shape, cur, mesh_sizes, md)
            locals_, cur = slice_dim(locals_, global_shape, cur, mesh_sizes, md, dst)
    return locals_, cur


def distribute(global_arr, placements, mesh_sizes):
    """Exact slices per coordinate; Partial keeps the value on coordinate 0 of
    each Partial dim and zeros elsewhere (placement.py:273-290)."""
    pdims = [i for i, p in enumerate(placements) if p[0] == "P"]
    out = {}
    for c in mesh_coords(mesh_sizes):
        idx = window(global_arr.shape, placements, mesh_sizes, c)
        loc = global_arr[np.ix_(*idx)].copy() if all(len(i) for i in idx) else \
            np.zeros([len(i) for i in idx], dtype=global_arr.dtype)
        if any(c[i] != 0 for i in pdims):
            loc = np.zeros_like(loc)
        out[c] = loc
    return out
