"""Random ops on torch tensors: fused sharded dropout with mask recomputation.

Mirrors the dropout call path of the reference -- ops.dropout (reference
/root/reference/pkg/src/spmdsim/ops.py:168-190) -> dispatch._execute's mask
branch (dispatch.py:567-576) -> rng.dropout_mask_local (rng.py:238-242) ->
engine.k_dropout_apply (engine.py:80-81) -- as ONE sm_100a kernel
(`sdr_dropout`) that draws the keep-mask and applies it in a single pass.

Backward regenerates the mask from the saved (seed, offset, THETA, window)
instead of storing it: gx = (g * m) * (1/(1-p)), the same
expression the reference's backward closure evaluates (ops.py:187-188).
"""

from __future__ import annotations

import ctypes as C
import math

import torch

from . import _lib, runtime as runtime_mod
from .placement import ShardView, full_view  # noqa: F401
from .rng import RngState, dtype_code

_DROP_TYPES = (torch.float32, torch.float64, torch.bfloat16, torch.float16)


def _check_p(status):
    if status == _lib.E_PARAM:
        return ValueError("dropout needs p in [0, 1)")
    if status == _lib.E_DTYPE:
        return TypeError("dtype not supported by dropout")
    return None


def _check_buffer(name: str, buf, x: torch.Tensor, dtypes: tuple):
    """A caller-supplied output/mask buffer the kernel writes through a raw
    pointer: it must match x's shape and device, be contiguous, and have one
    of `dtypes` -- anything else would be a silent wrong or out-of-bounds
    write."""
    if not isinstance(buf, torch.Tensor):
        raise TypeError(f"`{name}` must be a torch.Tensor, got {type(buf).__name__}")
    if buf.dtype not in dtypes:
        raise TypeError(f"`{name}` has dtype {buf.dtype}, expected one of {dtypes}")
    if tuple(buf.shape) != tuple(x.shape):
        raise ValueError(f"`{name}` has shape {tuple(buf.shape)}, x has {tuple(x.shape)}")
    if buf.device != x.device:
        raise ValueError(f"`{name}` is on {buf.device}, x is on {x.device}")
    if not buf.is_contiguous():
        raise ValueError(f"`{name}` must be contiguous")


def dropout_apply(x: torch.Tensor, p: float, state: RngState, view: ShardView | None = None, *,
                  out: torch.Tensor | None = None, out_dtype: torch.dtype | None = None,
                  mask: torch.Tensor | None = None) -> torch.Tensor:
    """One fused launch: y = (x * m) * (1/(1-p)) with m the keep-mask of
    Bernoulli(1-p) drawn at `state` over `view` (the window x holds; default:
    x is the whole tensor).  Does NOT advance `state`.

    out_dtype: x.dtype (default), or torch.float32 for a bfloat16 x -- the
    reference's own result dtype (ml_dtypes bf16 * Python float -> float32).
    mask: optional uint8/bool or x.dtype tensor receiving m."""
    if not 0.0 <= p < 1.0:
        raise ValueError(f"dropout needs p in [0, 1), got {p}")
    if x.dtype not in _DROP_TYPES:
        raise TypeError(f"dropout supports {_DROP_TYPES}, got {x.dtype}")
    if not x.is_cuda:
        raise ValueError("dropout runs on CUDA tensors only")
    view = full_view(tuple(x.shape)) if view is None else view
    if tuple(x.shape) != view.local_shape:
        raise ValueError(f"x has shape {tuple(x.shape)}, window is {view.local_shape}")
    x = x.contiguous()
    yd = x.dtype if out_dtype is None else out_dtype
    if yd != x.dtype and not (x.dtype == torch.bfloat16 and yd == torch.float32):
        raise TypeError(f"dropout of {x.dtype} produces {x.dtype} (or float32 for bfloat16), not {yd}")
    if out is None:
        out = torch.empty(x.shape, dtype=yd, device=x.device)
    else:
        _check_buffer("out", out, x, (yd,))
    mcode = -1
    if mask is not None:
        _check_buffer("mask", mask, x, (torch.uint8, torch.bool, x.dtype))
        mcode = dtype_code(mask.dtype)
    if x.numel() == 0:
        return out
    nr, nv = state.native(), view.to_native()
    if x.device.index == torch.cuda.current_device():
        st = _lib.LIB.sdr_dropout(x.data_ptr(), dtype_code(x.dtype), out.data_ptr(), dtype_code(yd),
                                  None if mask is None else mask.data_ptr(), mcode, float(p),
                                  C.byref(nr), C.byref(nv), _lib.stream_handle(x.device))
    else:
        with torch.cuda.device(x.device):
            st = _lib.LIB.sdr_dropout(x.data_ptr(), dtype_code(x.dtype), out.data_ptr(), dtype_code(yd),
                                      None if mask is None else mask.data_ptr(), mcode, float(p),
                                      C.byref(nr), C.byref(nv), _lib.stream_handle(x.device))
    _lib.check(st, "sdr_dropout", _check_p)
    return out


class _Dropout(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, p, state_tuple, view):
        st = RngState(*state_tuple)
        ctx.p, ctx.state_tuple, ctx.view = p, state_tuple, view
        return dropout_apply(x, p, st, view)

    @staticmethod
    def backward(ctx, g):
        gx = dropout_apply(g.contiguous(), ctx.p, RngState(*ctx.state_tuple), ctx.view)
        return gx, None, None, None


def dropout(x: torch.Tensor, p: float, state: RngState | None = None,
            view: ShardView | None = None, training: bool = True) -> torch.Tensor:
    """Dropout with single-device semantics (reference ops.py:168-190).

    `view` is the window of the global tensor that x holds (default: all of
    it); the mask is the slice of ONE global Bernoulli draw, so any sharding
    gives the same merged output.  p == 0 returns x and consumes no random
    numbers (ops.py:174-175); otherwise the state advances by
    ceil(global_numel / THETA) on every rank."""
    if not training or p == 0.0:
        return x
    state = runtime_mod.current().rng if state is None else state
    view = full_view(tuple(x.shape)) if view is None else view
    snap = (state.seed, state.offset, state.global_threads)
    if x.requires_grad and torch.is_grad_enabled():
        y = _Dropout.apply(x, p, snap, view)
    else:
        y = dropout_apply(x, p, state, view)
    state.advance(math.prod(view.global_shape))
    return y


# ---------------------------------------------------------------------------
# Dropout on a DTensor (dispatch.py:499-576 for op "dropout").
# ---------------------------------------------------------------------------
# Per-mesh-dim redistribution cost in multiples of S*(P-1)/P (dispatch.py:289-302).
_COST = {("S", "R"): 1, ("IS", "R"): 1, ("P", "R"): 2, ("P", "S"): 1, ("P", "IS"): 1,
         ("R", "S"): 0, ("R", "IS"): 0, ("S", "S"): 1, ("S", "IS"): 1, ("IS", "S"): 1,
         ("IS", "IS"): 1}


def _kind(p):
    from .placement import InterleavedShard, Partial, Shard
    if isinstance(p, Shard):
        return "S"
    if isinstance(p, InterleavedShard):
        return "IS"
    if isinstance(p, Partial):
        return "P"
    return "R"


def dropout_input_spec(x):
    """The placement dropout runs at: the cheapest (in bytes moved) spec among
    R / S(d) / the input's own IS per mesh dim -- Partial is not allowed --
    first in enumeration order on ties (dispatch.py:181-191, 330-372).  A
    Partial input therefore becomes a reduce-scatter to the first free S(d)."""
    import itertools
    from fractions import Fraction
    from .placement import InterleavedShard, PlacementError, Replicate, Shard, ShardSpec
    spec = x.meta.spec
    mesh = spec.mesh
    ndim = len(x.shape)
    choices = [Replicate()] + [Shard(d) for d in range(ndim)]
    choices += [p for p in spec.placements if isinstance(p, InterleavedShard) and p not in choices]
    nbytes = math.prod(x.shape) * x.local.element_size()
    best = None
    for combo in itertools.product(choices, repeat=mesh.ndim):
        try:
            cand = ShardSpec(mesh, tuple(combo))
            cand.validate_for_shape(x.shape)
        except PlacementError:
            continue
        cost = Fraction(0)
        ok = True
        for i, (s, d) in enumerate(zip(spec.placements, cand.placements)):
            if s == d:
                continue
            key = (_kind(s), _kind(d))
            if key not in _COST:
                ok = False
                break
            P = mesh.sizes[i]
            cost += _COST[key] * Fraction(nbytes * (P - 1), P)
        if ok and (best is None or cost < best[0]):
            best = (cost, cand)
    return best[1]


def dropout_plan_directive(site: str, x) -> str:
    """The static-plan directive the reference records for a dropout call
    site (dispatch.py:612-624): `annotate <site>.<in> <placements>`, naming the
    placement the mask is drawn at.  Replaying it (dtensor_dropout(at=...))
    draws the same global mask at the same placement."""
    from .placement import format_placements
    return f"annotate {site}.<in> {format_placements(dropout_input_spec(x).placements)}"


def dtensor_dropout(x, p: float, state: RngState | None = None, ledger=None, *, mover=None,
                    at=None):
    """Dropout of a DTensor with single-device semantics.  The mask is this
    rank's slice of ONE global Bernoulli(1-p) draw over the input window, the
    state advances by ceil(global_numel/THETA) on every rank (dispatch.py:
    567-576); p == 0 returns x untouched and draws nothing (ops.py:174-175).
    `at` (a ShardSpec) is the static-eager path: the placement a recorded
    plan annotated for this site (dispatch.py:604-608), instead of the
    dynamic choice."""
    from .dtensor import DTensor, redistribute
    if p == 0.0:
        return x
    state = runtime_mod.current().rng if state is None else state
    target = dropout_input_spec(x) if at is None else at
    if target != x.meta.spec:
        x = redistribute(x, target, ledger, mover=mover)
    y = dropout_apply(x.local, p, state, x.view)
    state.advance(math.prod(x.shape))
    return DTensor(x.meta, y, x.coord)


# ---------------------------------------------------------------------------
# Host-buffer dropout: pipelined H2D -> fused kernel -> D2H.
# ---------------------------------------------------------------------------
_PIPE: dict = {}
_PIPE_NBUF = 3  # device staging buffers per direction in dropout_host


def _pipe_state(device, nbytes_in, nbytes_out, dtype_in, dtype_out, nbuf):
    key = (device, dtype_in, dtype_out, nbuf)
    st = _PIPE.get(key)
    if st is None or st["cap_in"] < nbytes_in or st["cap_out"] < nbytes_out:
        if st is not None:  # in-flight (sync=False) work may still use the old buffers
            for k in ("h2d", "comp", "d2h"):
                st[k].synchronize()
        st = {"cap_in": nbytes_in, "cap_out": nbytes_out,
              "xin": [torch.empty(nbytes_in, dtype=torch.uint8, device=device) for _ in range(nbuf)],
              "yout": [torch.empty(nbytes_out, dtype=torch.uint8, device=device) for _ in range(nbuf)],
              "h2d": torch.cuda.Stream(device), "comp": torch.cuda.Stream(device),
              "d2h": torch.cuda.Stream(device),
              # per staging buffer: event after its last D2H (persists across calls so
              # back-to-back sync=False calls never overwrite a buffer still being read)
              "d2h_done": [None] * nbuf, "next": 0}
        _PIPE[key] = st
    return st


def _host_blocks(shape, view: ShardView, chunks: int):
    """Cut a window into contiguous product sub-windows for the host pipeline.
    The window is walked as R "rows" (dim-0 indices, or dim-0 x dim-1 indices
    when dim 1 is a plain range); blocks grow from R/chunks rows by doubling to
    R/8 and shrink the same way at the end, so the pipeline fill (first H2D)
    and drain (last D2H) are short while the middle needs few copies.  A block
    never straddles a dim-0 index unless it spans whole dim-0 rows.  Yields
    (index tuple, sub-view)."""
    from .placement import DimWindow
    wins = tuple(view.windows)
    if not shape or shape[0] == 0 or wins[0].groups != 1 or math.prod(shape) == 0:
        yield (slice(None),), view
        return
    L = shape[1] if len(shape) >= 2 and wins[1].groups == 1 and shape[1] >= 2 else 1
    R = shape[0] * L
    unit = max(1, R // max(1, chunks))
    big = max(unit, R // 8)
    head = []
    s = unit
    while sum(head) + s <= R // 2 and s < big:
        head.append(s)
        s *= 2
    H = sum(head)
    step = max(L, big // L * L) if L > 1 else big
    pts = {0, R}
    acc = 0
    for n in head:
        acc += n
        pts.update((acc, R - acc))
    pts.update(range(-(-H // step) * step, R - H, step))
    pts = sorted(p for p in pts if 0 <= p <= R)
    cuts = []
    for a, b in zip(pts, pts[1:]):
        while a < b:  # split at dim-0 boundaries unless spanning whole dim-0 rows
            if L > 1 and (a % L or b - a < L):
                e = min(b, (a // L + 1) * L)
            elif L > 1:
                e = b - b % L
            else:
                e = b
            cuts.append((a, e))
            a = e
    for a, b in cuts:
        if L == 1 or (a % L == 0 and b % L == 0):
            r0, r1 = a // L, b // L
            yield (slice(r0, r1),), ShardView(view.global_shape,
                                              windows=(DimWindow(wins[0].start + r0, r1 - r0),) + wins[1:])
        else:
            r, c0, c1 = a // L, a % L, b - (a // L) * L
            yield (slice(r, r + 1), slice(c0, c1)), ShardView(
                view.global_shape, windows=(DimWindow(wins[0].start + r, 1),
                                            DimWindow(wins[1].start + c0, c1 - c0)) + wins[2:])


def dropout_host(x_host: torch.Tensor, p: float, state: RngState, view: ShardView | None = None, *,
                 out: torch.Tensor | None = None, out_dtype: torch.dtype | None = None,
                 device=None, chunks: int = 16, sync: bool = True) -> torch.Tensor:
    """dropout_apply for a tensor in (pinned) HOST memory, result in host
    memory.  The window is cut into contiguous blocks of 1/chunks .. 1/8 of it
    (_host_blocks, tapered at both ends); block i's H2D copy, block i-1's fused kernel and block
    i-2's D2H copy run concurrently on three streams (PCIe is full duplex), so
    the end-to-end time approaches max(H2D, D2H) instead of their sum.  Values
    are identical to dropout_apply (each block is a sub-window of the same
    global draw).  Does NOT advance `state`.  With sync=True (default) it
    blocks the host until the result is ready; with sync=False it returns at
    once, stream-ordered after the caller's current stream (which waits for the
    result): consecutive calls then keep both PCIe directions busy across
    calls, like a prefetching input pipeline.  `x_host` must stay unchanged and
    `out` unread until the stream reaches that point."""
    if x_host.is_cuda:
        raise ValueError("dropout_host expects a host tensor; use dropout_apply for device tensors")
    view = full_view(tuple(x_host.shape)) if view is None else view
    if tuple(x_host.shape) != view.local_shape:
        raise ValueError(f"x has shape {tuple(x_host.shape)}, window is {view.local_shape}")
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    yd = x_host.dtype if out_dtype is None else out_dtype
    if out is None:
        out = torch.empty(x_host.shape, dtype=yd, pin_memory=True)
    else:
        _check_buffer("out", out, x_host, (yd,))
    x_host = x_host.contiguous()
    if x_host.dim() == 0:
        blocks = [((), view)]
    else:
        blocks = list(_host_blocks(tuple(x_host.shape), view, max(1, chunks)))
    cap = max(int(x_host[ix].numel()) for ix, _ in blocks) if x_host.dim() else 1
    nbuf = _PIPE_NBUF
    S = _pipe_state(dev, cap * x_host.element_size(), cap * torch.empty((), dtype=yd).element_size(),
                    x_host.dtype, yd, nbuf)
    cur = torch.cuda.current_stream(dev)
    d2h_done = S["d2h_done"]
    for s in (S["h2d"], S["comp"], S["d2h"]):
        s.wait_stream(cur)
    first = S["next"]
    S["next"] = (first + len(blocks)) % nbuf
    for i, (ix, sub) in enumerate(blocks):
        b = (first + i) % nbuf
        xs = x_host[ix]
        n = xs.numel()
        if n == 0:
            continue
        xin = S["xin"][b][:n * x_host.element_size()].view(x_host.dtype).view(xs.shape)
        yout = S["yout"][b][:n * out.element_size()].view(yd).view(xs.shape)
        h2d_done, comp_done = torch.cuda.Event(), torch.cuda.Event()
        with torch.cuda.stream(S["h2d"]):
            if d2h_done[b] is not None:
                S["h2d"].wait_event(d2h_done[b])  # buffer b free again
            xin.copy_(xs, non_blocking=True)
            h2d_done.record(S["h2d"])
        with torch.cuda.stream(S["comp"]):
            S["comp"].wait_event(h2d_done)
            dropout_apply(xin, p, state, sub, out=yout, out_dtype=yd)
            comp_done.record(S["comp"])
        with torch.cuda.stream(S["d2h"]):
            S["d2h"].wait_event(comp_done)
            out[ix].copy_(yout, non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(S["d2h"])
            d2h_done[b] = ev
    cur.wait_stream(S["d2h"])
    if sync:
        cur.synchronize()
    return out


# ---------------------------------------------------------------------------
# Traced redistribute (reference ops.py:193-217): a placement change whose
# backward sends the incoming gradient to `grad_spec` (default: the source
# placement with Partial flipped to Replicate -- a Partial forward value
# carries a replicated gradient).
# ---------------------------------------------------------------------------
class _RedistributeFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, local, x, dst, grad_spec, ledger):
        from .dtensor import DTensor
        from .dtensor import redistribute as dt_redistribute
        src = DTensor(x.meta, local, x.coord)
        y = dt_redistribute(src, dst, ledger)
        ctx.meta, ctx.coord, ctx.dst, ctx.grad_spec, ctx.ledger = y.meta, x.coord, dst, grad_spec, ledger
        return y.local

    @staticmethod
    def backward(ctx, g):
        from dataclasses import replace as _replace
        from .dtensor import DTensor
        from .dtensor import redistribute as dt_redistribute
        gd = DTensor(_replace(ctx.meta, dtype=g.dtype), g.contiguous(), ctx.coord)
        if ctx.dst != ctx.grad_spec:
            gd = dt_redistribute(gd, ctx.grad_spec, ctx.ledger)
        return gd.local, None, None, None, None


def redistribute(x, dst, grad_spec=None, ledger=None):
    """Differentiable placement change of a DTensor (reference ops.py:193-217):
    the forward is dtensor.redistribute; autograd on the local shard routes the
    gradient back to `grad_spec`.  A plain (non-DTensor) tensor is returned
    unchanged, as in the reference's single-device run."""
    from dataclasses import replace as _replace
    from .dtensor import DTensor
    from .placement import Partial, Replicate, ShardSpec
    if not isinstance(x, DTensor):
        return x
    if grad_spec is None:
        src = x.meta.spec
        grad_spec = ShardSpec(src.mesh, tuple(Replicate() if isinstance(p, Partial) else p
                                              for p in src.placements))
    local = _RedistributeFn.apply(x.local, x, dst, grad_spec, ledger)
    return DTensor(_replace(x.meta, spec=dst), local, x.coord)

