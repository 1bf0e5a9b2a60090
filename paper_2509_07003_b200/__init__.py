"""B200-native single-device-semantic distributed RNG + fused redistribute.

A from-scratch sm_100a implementation of veScale's (arXiv 2509.07003)
distributed-RNG hot path behind the Python API of the reference simulator
`spmdsim` (/root/reference/pkg/src/spmdsim/__init__.py:3-32).  All arithmetic
runs in `libsdrng.so` (hand-written CUDA for sm_100a, C ABI in
include/sdrng.h); collectives use NCCL through torch.distributed.
"""

from .mesh import DeviceMesh, MeshError, create_mesh
from .placement import (
    InterleavedShard,
    Partial,
    Placement,
    PlacementError,
    Replicate,
    Shard,
    ShardSpec,
    ShardView,
    full_view,
    local_shape_and_offset,
    parse_placements,
)
from .rng import (
    Bernoulli,
    Normal,
    RandInt,
    RngState,
    Uniform,
    Uniform01,
    dropout_mask_local,
    fill_random,
    generate_distributed,
    generate_global,
    generate_local,
)
from .ops import dropout
from .dtensor import DTensor, DTensorMeta, distribute, from_local, redistribute, redistribute_many, to_global

__all__ = [
    "DeviceMesh", "MeshError", "create_mesh",
    "Placement", "Shard", "Replicate", "Partial", "InterleavedShard", "ShardSpec", "ShardView",
    "PlacementError", "full_view", "local_shape_and_offset", "parse_placements",
    "RngState", "Uniform01", "Uniform", "Normal", "RandInt", "Bernoulli",
    "fill_random", "generate_global", "generate_distributed", "generate_local",
    "dropout_mask_local", "dropout",
    # reference top-level exports (spmdsim/__init__.py:3-32)
    "DTensor", "DTensorMeta", "distribute", "redistribute", "to_global",
    "from_local", "redistribute_many",
]
