"""Device topology: an N-d mesh over global ranks, its fibers and flattenings.

API mirror of spmdsim.mesh (reference: /root/reference/pkg/src/spmdsim/
mesh.py:20-172).  Ranks are laid out row-major over the named dimensions, so a
rank's coordinates are the mixed-radix digits of its position in `ranks`.
In the multi-process build every process owns one rank (one GPU); the fiber
sub-groups used by collectives are created by `paper_2509_07003_b200.comm`.
"""

from __future__ import annotations

import itertools
import math
from dataclasses import dataclass


class MeshError(ValueError):
    """Bad mesh construction or lookup (reference mesh.py:16-17)."""


def _digits(index: int, radices) -> tuple[int, ...]:
    out = [0] * len(radices)
    for pos in range(len(radices) - 1, -1, -1):
        index, out[pos] = divmod(index, radices[pos])
    return tuple(out)


def _linear(digits, radices) -> int:
    idx = 0
    for d, r in zip(digits, radices):
        idx = idx * r + d
    return idx


@dataclass(frozen=True)
class DeviceMesh:
    """Named dimensions (name, size) over an ordered rank list (row-major)."""
    name: str
    dims: tuple[tuple[str, int], ...]
    ranks: tuple[int, ...]

    def __post_init__(self):
        labels, radices = zip(*self.dims) if self.dims else ((), ())
        checks = [
            (not radices, "a mesh needs at least one dimension"),
            (bool(radices) and min(radices) < 1, f"every mesh dimension must have size >= 1, got {list(radices)}"),
            (math.prod(radices) != len(self.ranks), f"{len(self.ranks)} ranks cannot fill sizes {list(radices)}"),
            (len(set(self.ranks)) < len(self.ranks), "a rank appears twice in the mesh"),
            (len(set(labels)) < len(labels), f"mesh dimension names repeat: {list(labels)}"),
        ]
        for bad, msg in checks:
            if bad:
                raise MeshError(msg)

    # shape ---------------------------------------------------------------------
    ndim = property(lambda self: len(self.dims))
    sizes = property(lambda self: tuple(sz for _, sz in self.dims))
    dim_names = property(lambda self: tuple(nm for nm, _ in self.dims))

    def size(self) -> int:
        """Number of devices."""
        return len(self.ranks)

    def dim_index(self, dim_name: str) -> int:
        for i, (nm, _) in enumerate(self.dims):
            if nm == dim_name:
                return i
        raise MeshError(f"no mesh dimension {dim_name!r} among {self.dim_names}")

    def dim_size(self, dim_name: str) -> int:
        return self.dims[self.dim_index(dim_name)][1]

    # -- coordinates -----------------------------------------------------------
    def coords_of_rank(self, rank: int) -> tuple[int, ...]:
        if rank not in self.ranks:
            raise MeshError(f"rank {rank} is not part of mesh {self.name}")
        return _digits(self.ranks.index(rank), self.sizes)

    def rank_at(self, coords) -> int:
        coords = tuple(coords)
        if len(coords) != self.ndim:
            raise MeshError(f"coordinate {coords} does not address a {self.ndim}-d mesh")
        if any(not 0 <= c < s for c, s in zip(coords, self.sizes)):
            raise MeshError(f"coordinate {coords} is outside mesh sizes {self.sizes}")
        return self.ranks[_linear(coords, self.sizes)]

    def iter_coords(self):
        """Every coordinate in ascending row-major order."""
        return itertools.product(*[range(s) for s in self.sizes])

    # -- sub-meshes --------------------------------------------------------------
    def fiber_ranks(self, dim_indices, fixed_coords) -> list[int]:
        """Ranks of the fiber spanned by `dim_indices` through `fixed_coords`
        (row-major over the spanned dims)."""
        spans = [range(self.sizes[d]) if d in dim_indices else (fixed_coords[d],)
                 for d in range(self.ndim)]
        return [self.rank_at(c) for c in itertools.product(*spans)]

    def submesh(self, dim_name: str, rank: int) -> "DeviceMesh":
        """The 1-d fiber along `dim_name` that contains `rank`."""
        d = self.dim_index(dim_name)
        members = self.fiber_ranks((d,), self.coords_of_rank(rank))
        return DeviceMesh(f"{self.name}.{dim_name}", ((dim_name, self.sizes[d]),), tuple(members))

    def fibers(self, dim_indices) -> list[list[int]]:
        """All fibers spanned by `dim_indices`, in ascending order of the fixed
        coordinates (the order every rank must create process groups in)."""
        dim_indices = tuple(sorted(dim_indices))
        rest = [d for d in range(self.ndim) if d not in dim_indices]
        out = []
        for fixed in itertools.product(*[range(self.sizes[d]) for d in rest]):
            full = [0] * self.ndim
            for d, c in zip(rest, fixed):
                full[d] = c
            out.append(self.fiber_ranks(dim_indices, full))
        return out

    def flatten_dims(self, dim_names, new_name: str | None = None) -> "DeviceMesh":
        """Merge the named dims into one dimension placed where the first of
        them sits, ordered row-major over the merged coordinates in
        declaration order (reference mesh.py:119-162)."""
        if not dim_names:
            raise MeshError("flatten_dims needs at least one dimension name")
        picked = [self.dim_index(n) for n in dim_names]
        if len(set(picked)) != len(picked):
            raise MeshError(f"dimension named twice in {list(dim_names)}")
        picked = sorted(picked)
        merged_size = math.prod(self.sizes[d] for d in picked)
        merged_name = new_name or "_".join(self.dim_names[d] for d in picked)
        new_dims = []
        for d in range(self.ndim):
            if d == picked[0]:
                new_dims.append((merged_name, merged_size))
            elif d not in picked:
                new_dims.append(self.dims[d])
        merged_pos = picked[0]  # every dim before it is kept, so its index is unchanged
        kept = [d for d in range(self.ndim) if d not in picked]
        picked_sizes = [self.sizes[d] for d in picked]
        ranks = []
        for nc in itertools.product(*[range(s) for _, s in new_dims]):
            old = [0] * self.ndim
            kept_it = iter(kept)
            for pos, c in enumerate(nc):
                if pos == merged_pos:
                    for d, dig in zip(picked, _digits(c, picked_sizes)):
                        old[d] = dig
                else:
                    old[next(kept_it)] = c
            ranks.append(self.rank_at(old))
        return DeviceMesh(f"{self.name}.flat({merged_name})", tuple(new_dims), tuple(ranks))


def create_mesh(dims, ranks=None, name: str = "mesh") -> DeviceMesh:
    """Row-major mesh over `ranks`, default 0..N-1 (reference mesh.py:165-172)."""
    spec = tuple((str(label), int(extent)) for label, extent in dims)
    order = tuple(range(math.prod(e for _, e in spec))) if ranks is None else tuple(map(int, ranks))
    return DeviceMesh(name=name, dims=spec, ranks=order)
