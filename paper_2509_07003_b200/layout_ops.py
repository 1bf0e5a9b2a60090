"""Whole-tensor layout helpers: split a full tensor into every coordinate's
shard and merge shards back (torch; single process).  API of the reference's
placement.distribute_local_tensors / merge_local_tensors (reference:
/root/reference/pkg/src/spmdsim/placement.py:273-355): Partial dims merge by a
sum in ascending coordinate order, Replicate copies must agree bit for bit.
"""

from __future__ import annotations

import torch

from .placement import PlacementError, ShardSpec, local_shape_and_offset


def _gather_window(t: torch.Tensor, view):
    if not view.num_local_elements:
        return t.new_zeros(view.local_shape)
    grids = torch.meshgrid(*[torch.as_tensor(ix, device=t.device) for ix in view.index_lists],
                           indexing="ij")
    return t[grids].clone()


def distribute_local_tensors(spec: ShardSpec, global_tensor) -> dict:
    """Exact per-coordinate slices (torch); Partial keeps the value on
    coordinate 0 of every Partial dim, zeros elsewhere (placement.py:273-290)."""
    spec.validate_for_shape(tuple(global_tensor.shape))
    pdims = spec.partial_mesh_dims()
    out = {}
    for coord in spec.mesh.iter_coords():
        loc = _gather_window(global_tensor, local_shape_and_offset(spec, tuple(global_tensor.shape), coord))
        if any(coord[d] for d in pdims):
            loc = torch.zeros_like(loc)
        out[coord] = loc
    return out


def _bits(t):
    return t.contiguous().reshape(-1).view(torch.uint8)


def merge_local_tensors(spec: ShardSpec, global_shape, locals_: dict):
    """Inverse of distribute_local_tensors (torch): Partial dims are summed in
    ascending coordinate order, Replicate copies must be bit-identical
    (placement.py:293-355)."""
    spec.validate_for_shape(global_shape)
    mesh = spec.mesh
    coords = list(mesh.iter_coords())
    if set(locals_) != set(coords):
        raise PlacementError("locals must cover every mesh coordinate exactly once")
    pdims = spec.partial_mesh_dims()
    sdims = [i for i, p in enumerate(spec.placements) if p.is_shard_like()]
    summed: dict = {}
    for coord in coords:
        view = local_shape_and_offset(spec, global_shape, coord)
        loc = locals_[coord]
        if tuple(loc.shape) != view.local_shape:
            raise PlacementError(f"local at {coord} has shape {tuple(loc.shape)}, expected {view.local_shape}")
        key = tuple(c for i, c in enumerate(coord) if i not in pdims)
        summed[key] = loc.clone() if key not in summed else summed[key] + loc
    first = next(iter(locals_.values()))
    out = torch.zeros(tuple(global_shape), dtype=first.dtype, device=first.device)
    seen: dict = {}
    nonpartial = [i for i in range(mesh.ndim) if i not in pdims]
    for key, loc in summed.items():
        skey = tuple(c for i, c in zip(nonpartial, key) if i in sdims)
        if skey in seen:
            ref = seen[skey]
            if ref.shape != loc.shape or not torch.equal(_bits(ref), _bits(loc)):
                raise PlacementError(f"replica mismatch at shard coordinate {skey}")
            continue
        seen[skey] = loc
        coord = [0] * mesh.ndim
        for i, c in zip(sdims, skey):
            coord[i] = c
        view = local_shape_and_offset(spec, global_shape, tuple(coord))
        if view.num_local_elements:
            idx = [torch.as_tensor(ix, device=out.device) for ix in view.index_lists]
            out[torch.meshgrid(*idx, indexing="ij")] = loc
    return out
