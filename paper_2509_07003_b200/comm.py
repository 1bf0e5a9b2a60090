"""Collectives over NCCL process groups, byte ledger, bucketing and N-d fusion.

API mirror of spmdsim.comm (reference: /root/reference/pkg/src/spmdsim/
comm.py:1-318).  The reference simulates every device in one process and sums
in ascending rank order; here each process is one rank (one B200) and the
collectives are NCCL calls on per-fiber process groups.  The ledger keeps the
reference's ring byte model (comm.py:45-62), which is also the NCCL-tests
bus-bandwidth convention used by bench.py.
"""

from __future__ import annotations

import os

from dataclasses import dataclass, field
from fractions import Fraction

from .ledger import CollectiveLedger, LedgerEntry  # noqa: F401  (API re-export)

DEFAULT_BUCKET_BYTES = 65536


class CommError(ValueError):
    pass


# ---------------------------------------------------------------------------
# Process groups: one per fiber of each (set of) mesh dim(s).
# ---------------------------------------------------------------------------
_GROUPS: dict = {}


def my_rank() -> int:
    import torch.distributed as dist
    return dist.get_rank() if dist.is_initialized() else 0


def fiber_group(mesh, dims: tuple):
    """(process group, fiber ranks in coordinate order) of this rank's fiber
    spanned by mesh dims `dims` (several dims = the flattened N-d fiber,
    mesh.flatten_dims order).  Every rank creates every fiber group of `dims`
    in the same order on first use, as torch.distributed requires."""
    import torch.distributed as dist
    key = (mesh, tuple(dims))
    if key not in _GROUPS:
        me = my_rank()
        mine = None
        fibers = mesh.fibers(tuple(dims))
        for fib in fibers:
            if fib != sorted(fib):
                raise CommError(f"fiber {fib} is not in ascending rank order; "
                                "build the mesh with row-major ranks")
            g = dist.new_group(ranks=fib) if (dist.is_initialized() and len(fib) > 1) else None
            if me in fib:
                mine = (g, fib)
        if mine is None:
            raise CommError(f"rank {me} is not in mesh {mesh.name}")
        _GROUPS[key] = mine
    return _GROUPS[key]


def _host_staged(t) -> bool:
    """Test hook (SDR_COMM_CPU_STAGING=1): CUDA buffers cross a gloo group via
    host copies, so several processes sharing one GPU can run the CUDA movers
    end to end.  Never set in production (NCCL moves device buffers)."""
    return t.is_cuda and os.environ.get("SDR_COMM_CPU_STAGING") == "1"


def all_gather_into(recv, send, group, ledger=None, mesh="", dims="", P=1, nbytes=None):
    """recv[P*len(send)] <- every fiber member's `send`, in fiber order.
    `nbytes` is the payload the ledger records (default: recv's bytes); a
    coalesced call passes its members' real bytes, without padding."""
    import torch.distributed as dist
    if P == 1 or group is None:
        recv.copy_(send)
    elif _host_staged(recv):
        r = recv.cpu()
        dist.all_gather_into_tensor(r, send.cpu(), group=group)
        recv.copy_(r)
    else:
        dist.all_gather_into_tensor(recv, send, group=group)
    if ledger is not None:
        ledger.record("all_gather", recv.numel() * recv.element_size() if nbytes is None else nbytes,
                      P, mesh, dims)


def reduce_scatter_into(out, inp, group, ledger=None, mesh="", dims="", P=1, nbytes=None):
    """out <- this rank's segment of the elementwise sum of every member's inp
    (`nbytes`: the ledger payload, as in all_gather_into)."""
    import torch.distributed as dist
    if P == 1 or group is None:
        out.copy_(inp)
    elif _host_staged(out):
        o = out.cpu()
        dist.reduce_scatter_tensor(o, inp.cpu(), op=dist.ReduceOp.SUM, group=group)
        out.copy_(o)
    else:
        dist.reduce_scatter_tensor(out, inp, op=dist.ReduceOp.SUM, group=group)
    if ledger is not None:
        ledger.record("reduce_scatter", inp.numel() * inp.element_size() if nbytes is None else nbytes,
                      P, mesh, dims)


def all_reduce_into(buf, group, ledger=None, mesh="", dims="", P=1, nbytes=None):
    import torch.distributed as dist
    if P > 1 and group is not None and _host_staged(buf):
        b = buf.cpu()
        dist.all_reduce(b, op=dist.ReduceOp.SUM, group=group)
        buf.copy_(b)
    elif P > 1 and group is not None:
        dist.all_reduce(buf, op=dist.ReduceOp.SUM, group=group)
    if ledger is not None:
        ledger.record("all_reduce", buf.numel() * buf.element_size() if nbytes is None else nbytes,
                      P, mesh, dims)


# ---------------------------------------------------------------------------
# Bucketed and N-dim fused gradient reduction (comm.py:130-289).
# ---------------------------------------------------------------------------
# ---------------------------------------------------------------------------
# Single-process collectives over per-participant tensors (reference
# comm.py:91-125): the simulator's forms, kept for drop-in code that builds
# every coordinate's buffer in one process.  Sums run in ascending group-rank
# order on the tensors' device, exactly like the reference.
# ---------------------------------------------------------------------------
def all_reduce(buffers, ledger=None, mesh: str = "", dims: str = ""):
    """Sum in ascending group-rank order; every participant gets the result."""
    shapes = {tuple(b.shape) for b in buffers}
    if len(shapes) != 1:
        raise CommError(f"all_reduce buffer shape mismatch: {shapes}")
    acc = buffers[0].clone()
    for b in buffers[1:]:
        acc += b
    if ledger is not None:
        ledger.record("all_reduce", buffers[0].numel() * buffers[0].element_size(), len(buffers), mesh, dims)
    return acc


def all_gather(shards, ledger=None, mesh: str = "", dims: str = ""):
    """Every participant receives the full shard list, in group-rank order."""
    if ledger is not None:
        ledger.record("all_gather", sum(s.numel() * s.element_size() for s in shards), len(shards), mesh, dims)
    return list(shards)


def reduce_scatter(buffers, slicer, ledger=None, mesh: str = "", dims: str = ""):
    """Sum in ascending group-rank order, then hand participant k slicer(sum, k)."""
    shapes = {tuple(b.shape) for b in buffers}
    if len(shapes) != 1:
        raise CommError(f"reduce_scatter buffer shape mismatch: {shapes}")
    acc = buffers[0].clone()
    for b in buffers[1:]:
        acc += b
    if ledger is not None:
        ledger.record("reduce_scatter", buffers[0].numel() * buffers[0].element_size(), len(buffers), mesh, dims)
    return [slicer(acc, k) for k in range(len(buffers))]


@dataclass
class GradBucket:
    """One greedy gradient bucket (reference comm.py:131-138)."""
    capacity_bytes: int
    members: list = field(default_factory=list)  # DTensor refs
    member_bytes: int = 0

    def fits(self, nbytes: int) -> bool:
        return not self.members or self.member_bytes + nbytes <= self.capacity_bytes


def bucketize(tensors, capacity_bytes: int) -> list[list]:
    """Greedy buckets over the REVERSED creation order (gradients become ready
    back to front); a tensor larger than the capacity gets a bucket of its
    own (reference comm.py:140-150).  Sizes are the largest local shard over
    the mesh (local_nbytes_max, as the reference's _pack_buckets): derived
    from the spec alone, so every rank -- in every fiber -- cuts the same
    buckets even for uneven shards."""
    out: list[list] = []
    used = 0
    for t in tensors[::-1]:
        nb = t.local_nbytes_max()
        if not out or (used + nb > capacity_bytes and out[-1]):
            out.append([])
            used = 0
        out[-1].append(t)
        used += nb
    return out


def _group_by_partial(grads):
    """{(mesh, partial mesh dims, dtype): [grads]} and the grads without a
    Partial dim (reference comm.py:153-164, plus dtype: one NCCL dtype per call)."""
    groups: dict = {}
    untouched = []
    for g in grads:
        dims = g.meta.spec.partial_mesh_dims()
        if dims:
            groups.setdefault((g.meta.spec.mesh, dims, g.dtype), []).append(g)
        else:
            untouched.append(g)
    return groups, untouched


REDUCE_MODES = ("exact", "switch")


def reduce_mode(mode: str | None = None) -> str:
    """How the P->R all-reduces of the gradient reductions sum.

    "exact" (default): the peer-memory pull, ascending fiber-rank order --
    bit-identical to the reference's `acc += b` loop (comm.py:91-101) for every
    dtype.  "switch" (opt-in; argument or SDR_PR_REDUCE=switch): one NCCL
    all-reduce per bucket over the flattened fiber communicator, which NCCL
    runs as NVLS -- the reduction inside the NVSwitch (multimem ld_reduce) --
    on nodes whose fabric supports it (NCCL_ALGO=NVLS forces it).  The
    switch's summation order is not the ascending rank order, so float
    results differ from the reference within `switch_sum_tolerance`;
    integer sums stay exact."""
    m = os.environ.get("SDR_PR_REDUCE", "exact") if mode is None else mode
    if m not in REDUCE_MODES:
        raise CommError(f"reduce mode must be one of {REDUCE_MODES}, not {m!r}")
    return m


def switch_sum_tolerance(abs_sum, P: int, dtype):
    """Elementwise bound on |s_switch - s_ref| for a sum of P terms whose
    absolute values sum to `abs_sum`, the two sums taken in any two orders
    with round-to-nearest in `dtype`: each is within gamma_(P-1) * abs_sum of
    the exact sum (Higham, Accuracy and Stability, eq. 4.4), so their
    difference is within 2 gamma_(P-1) abs_sum, gamma_n = n u / (1 - n u),
    u = 2^-(mantissa bits + 1).  Zero for integer dtypes."""
    import torch
    if not dtype.is_floating_point:
        return 0 * abs_sum
    u = {torch.float64: 2.0 ** -53, torch.float32: 2.0 ** -24, torch.bfloat16: 2.0 ** -8,
         torch.float16: 2.0 ** -11}[dtype]
    n = max(P - 1, 0)
    return abs_sum * (2.0 * n * u / (1.0 - n * u))


def _reduce_buckets(members, dims, bucket_bytes, ledger, mover, rounds, label, mode="exact"):
    from .dtensor import DTensor, _fused_all_reduce
    from .placement import Replicate
    from dataclasses import replace
    mesh = members[0].meta.spec.mesh
    out = {}
    for bucket in bucketize(members, bucket_bytes):
        slots = [[m.meta.spec, m.local] for m in bucket]
        _fused_all_reduce(mesh, dims, list(zip(bucket, slots)), ledger, mover, ledger_mesh=label,
                          switch=mode == "switch")
        rounds.append(("all_reduce", label, tuple(mesh.dim_names[d] for d in dims)))
        for m, (spec, loc) in zip(bucket, slots):
            for d in dims:
                spec = spec.with_placement(d, Replicate())
            out[id(m)] = DTensor(replace(m.meta, spec=spec), loc, m.coord)
    return out


def bucketed_grad_reduce(grads, bucket_bytes: int = DEFAULT_BUCKET_BYTES, ledger=None, *,
                         mover=None, reduce: str | None = None):
    """Per Partial mesh dim, one all-reduce per bucket (comm.py:208-233).
    `reduce`: "exact" (default) or "switch" (see reduce_mode)."""
    from .movers import DEFAULT_MOVER
    mover = DEFAULT_MOVER if mover is None else mover
    mode = reduce_mode(reduce)
    groups, skipped = _group_by_partial(grads)
    result = {id(g): g for g in grads}
    rounds: list = []
    for (mesh, pdims, _), members in groups.items():
        current = members
        for d in pdims:
            upd = _reduce_buckets(current, (d,), bucket_bytes, ledger, mover, rounds, mesh.name, mode)
            current = [upd[id(m)] for m in current]
        for before, after in zip(members, current):
            result[id(before)] = after
    return [result[id(g)] for g in grads], {"skipped": skipped, "rounds": rounds, "reduce": mode}


def fused_nd_grad_reduce(grads, bucket_bytes: int = DEFAULT_BUCKET_BYTES, ledger=None, *,
                         mover=None, reduce: str | None = None):
    """All Partial dims of a group flattened into one fiber: ONE all-reduce
    per bucket instead of one per dim (comm.py:236-289).
    `reduce="switch"` (or SDR_PR_REDUCE=switch) sends each bucket through
    NCCL on the flattened communicator -- in-switch NVLS reduction where the
    fabric has it -- instead of the bit-exact peer pull (reduce_mode)."""
    from .movers import DEFAULT_MOVER
    mover = DEFAULT_MOVER if mover is None else mover
    mode = reduce_mode(reduce)
    groups, skipped = _group_by_partial(grads)
    result = {id(g): g for g in grads}
    rounds: list = []
    for (mesh, pdims, _), members in groups.items():
        flat = mesh.flatten_dims([mesh.dim_names[d] for d in pdims])
        upd = _reduce_buckets(members, tuple(pdims), bucket_bytes, ledger, mover, rounds, flat.name, mode)
        for m in members:
            result[id(m)] = upd[id(m)]
    return [result[id(g)] for g in grads], {"skipped": skipped, "rounds": rounds, "reduce": mode}


@dataclass(frozen=True)
class CostParams:
    payload_bytes: int
    transfer_time_per_byte: Fraction
    device_counts: tuple

    def __post_init__(self):
        if self.payload_bytes <= 0 or self.transfer_time_per_byte <= 0:
            raise CommError("S and B must be positive")
        if not self.device_counts or any(p < 1 for p in self.device_counts):
            raise CommError("device counts must be >= 1")


def cost_model_eval(params: CostParams):
    """(T_vanilla, T_fused, ratio) of the ring model (comm.py:307-318)."""
    import math as _m
    two_sb = 2 * params.payload_bytes * Fraction(params.transfer_time_per_byte)
    tv = two_sb * sum(Fraction(p - 1, p) for p in params.device_counts)
    n = _m.prod(params.device_counts)
    tf = two_sb * Fraction(n - 1, n)
    return tv, tf, (tv / tf if tf else Fraction(1))
