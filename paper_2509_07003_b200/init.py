"""Deferred, shard-local parameter initialisation in ONE kernel launch.

Mirrors the reference's deferred init (reference: /root/reference/pkg/src/
spmdsim/model.py:21-46 Parameter.materialize_{global,sharded}, :121-132
Module.materialize, plan.py:280-290 parallelize -> materialize): parameters
record their initializer; materialisation walks them in DEFINITION ORDER, each
consuming ceil(numel/THETA) of the shared offset, and every rank fills only its
own shard.  Here the whole walk is one `sdr_fill_batch` launch: offsets are a
host prefix sum, the per-parameter windows/distributions go to the device as a
descriptor table, and CTAs tile all parameters (libsdrng K3).

The result is bit-identical to calling `generate_distributed` /
`generate_global` parameter by parameter (tests/test_init_gpu.py).
"""

from __future__ import annotations

import ctypes as C
import functools
import math
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .placement import ShardSpec, full_view, local_shape_and_offset
from .rng import Distribution, RngState, _TORCH_OF_CODE, _device, _note_allocation, _param_error, \
    dtype_code, ensure_normal_tables


@dataclass
class Parameter:
    """A named weight with a recorded initializer (model.py:21-46)."""
    shape: tuple
    dist: Distribution
    dtype: object = np.float64
    requires_grad: bool = True
    value: torch.Tensor | None = field(default=None, repr=False)

    def __post_init__(self):
        self.shape = tuple(int(n) for n in self.shape)

    @property
    def materialized(self) -> bool:
        return self.value is not None

    def materialize_global(self, state: RngState, *, device=None) -> torch.Tensor:
        """Single-device eager init: the full global tensor (model.py:36-39);
        advances `state` once."""
        from .rng import generate_global
        self.value = generate_global(self.shape, state, self.dist, self.dtype, device=device)
        return self.value

    def materialize_sharded(self, spec: ShardSpec, state: RngState, coord=None, *, device=None):
        """Local-only init (model.py:41-46): this rank fills just its own shard
        of the one global draw; advances `state` once.  Returns the DTensor
        (the local shard is also kept in `value`)."""
        from .dtensor import from_local
        from .rng import generate_local
        if coord is None:
            import torch.distributed as dist_mod
            rank = dist_mod.get_rank() if dist_mod.is_initialized() else 0
            coord = spec.mesh.coords_of_rank(rank)
        self.value = generate_local(spec, self.shape, state, self.dist, self.dtype, tuple(coord), device=device)
        return from_local(self.value, spec, self.shape, tuple(coord))


@functools.lru_cache(maxsize=4096)
def _window(spec: ShardSpec, shape: tuple, coord: tuple):
    """local_shape_and_offset, memoised: a model re-initialised (or many models
    with the same layout) recomputes no windows (ShardSpec is frozen/hashable)."""
    return local_shape_and_offset(spec, shape, coord)


def materialize(params, state: RngState, init_specs: dict | None = None, coord=None, *,
                device=None) -> dict:
    """Fill every not-yet-materialised parameter of `params` (an ordered
    mapping name -> Parameter, definition order) with ONE launch.

    init_specs maps name -> ShardSpec (absent = full tensor, like
    materialize_global); `coord` is this rank's mesh coordinate (default: the
    torch.distributed rank's).  Advances `state` exactly as the reference's
    sequential walk does.  Returns {name: local tensor}."""
    init_specs = init_specs or {}
    dev = _device(device)
    todo = [(n, p) for n, p in params.items() if not p.materialized]
    n = len(todo)
    if n == 0:
        return {}
    outs = (C.c_void_p * n)()
    dts = (C.c_int32 * n)()
    dists = (_lib.SdrDist * n)()
    rngs = (_lib.SdrRng * n)()
    views = (_lib.SdrView * n)()
    result = {}
    offset = state.offset
    need_normal = False
    for i, (name, p) in enumerate(todo):
        spec: ShardSpec | None = init_specs.get(name)
        if spec is None:
            view = full_view(p.shape)
        else:
            c = coord
            if c is None:
                import torch.distributed as dist_mod
                rank = dist_mod.get_rank() if dist_mod.is_initialized() else 0
                c = spec.mesh.coords_of_rank(rank)
            view = _window(spec, tuple(p.shape), tuple(c))
        code = p.dist.out_code(dtype_code(p.dtype))
        t = torch.empty(view.local_shape, dtype=_TORCH_OF_CODE[code], device=dev)
        result[name] = t
        outs[i] = t.data_ptr() if t.numel() else None
        dts[i] = code
        dists[i] = p.dist.native()
        rngs[i] = RngState(state.seed, offset, state.global_threads).native()
        views[i] = view.to_native()
        need_normal |= p.dist.kind == _lib.NORMAL
        offset += -(-math.prod(p.shape) // state.global_threads) * p.dist.blocks_per_element
    if need_normal:
        with torch.cuda.device(dev):
            ensure_normal_tables(dev)
    with torch.cuda.device(dev):
        st = _lib.LIB.sdr_fill_batch(outs, dts, dists, rngs, views, n, _lib.stream_handle(dev))
    _lib.check(st, "sdr_fill_batch", _param_error)
    for t in result.values():  # one fill per parameter, as the sequential walk records (rng.py:204)
        _note_allocation(t.numel())
    state.offset = offset
    for name, p in todo:
        p.value = result[name]
    return result


def llama3_8b_params(dist_factory, dtype="bfloat16") -> dict:
    """The 291 parameters of Meta-Llama-3-8B in HF definition order (embed,
    32 x {q,k,v,o,gate,up,down, 2 norms}, final norm, lm_head), each with the
    initializer `dist_factory(name, shape)`."""
    d, ff, kv, vocab, layers = 4096, 14336, 1024, 128256, 32
    shapes = [("model.embed_tokens.weight", (vocab, d))]
    for i in range(layers):
        pre = f"model.layers.{i}."
        shapes += [(pre + "self_attn.q_proj.weight", (d, d)),
                   (pre + "self_attn.k_proj.weight", (kv, d)),
                   (pre + "self_attn.v_proj.weight", (kv, d)),
                   (pre + "self_attn.o_proj.weight", (d, d)),
                   (pre + "mlp.gate_proj.weight", (ff, d)),
                   (pre + "mlp.up_proj.weight", (ff, d)),
                   (pre + "mlp.down_proj.weight", (d, ff)),
                   (pre + "input_layernorm.weight", (d,)),
                   (pre + "post_attention_layernorm.weight", (d,))]
    shapes += [("model.norm.weight", (d,)), ("lm_head.weight", (vocab, d))]
    return {n: Parameter(s, dist_factory(n, s), dtype) for n, s in shapes}


def llama3_tp_specs(params: dict, mesh, tp_dim: int = 0) -> dict:
    """TP placements of config 4: q,k,v,gate,up,embed,lm_head Shard(0);
    o,down Shard(1); norms Replicate (on the mesh dim `tp_dim`)."""
    from .placement import Replicate, Shard
    specs = {}
    for name, p in params.items():
        pl = [Replicate() for _ in range(mesh.ndim)]
        if len(p.shape) == 1:
            pass
        elif any(k in name for k in ("o_proj", "down_proj")):
            pl[tp_dim] = Shard(1)
        else:
            pl[tp_dim] = Shard(0)
        specs[name] = ShardSpec(mesh, tuple(pl))
    return specs


def materialize_module(module, init_fn, state: RngState, init_specs: dict | None = None, coord=None,
                       *, device=None) -> dict:
    """Deferred init of a torch.nn.Module built on the meta device (SURVEY
    8(f).2; reference plan.parallelize -> model.materialize, plan.py:280-290,
    model.py:121-132).  Parameters are taken in module.named_parameters() order
    (registration order, the reference's definition order); init_fn(name, p)
    returns the Distribution of each; init_specs maps name -> ShardSpec.  All
    parameters are filled by ONE launch and replaced in the module by their
    local shards (on `device`).  Returns {name: (global_shape, spec or None)}."""
    import torch.nn as nn
    table = {}
    for name, p in module.named_parameters():
        table[name] = Parameter(tuple(p.shape), init_fn(name, p), p.dtype, p.requires_grad)
    locals_ = materialize(table, state, init_specs, coord, device=device)
    owners = dict(module.named_modules())
    meta = {}
    for name, t in locals_.items():
        mod_name, _, leaf = name.rpartition(".")
        owner = owners[mod_name] if mod_name else module
        owner._parameters[leaf] = nn.Parameter(t, requires_grad=table[name].requires_grad)
        meta[name] = (table[name].shape, (init_specs or {}).get(name))
    return meta
