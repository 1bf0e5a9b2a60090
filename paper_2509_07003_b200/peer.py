"""Peer-memory transport for the coalesced redistribute collectives.

On an NVLink / NVSwitch node every rank of a fiber can load from every other
rank's HBM.  A `PeerHeap` is one CUDA-IPC-exported allocation per rank and
fiber (flag words + two data halves) mapped by all fiber ranks.  A coalesced
collective then runs as three launches on the current stream, with no NCCL
call and no host synchronisation:

    pack my members into my half h   (sdr_pack_local / sdr_pack_scatter)
    sdr_peer_barrier(epoch)          (release my flag, acquire everyone's)
    ONE pull kernel                  (sdr_unpack_gathered_peers: S->R, or
                                      sdr_reduce_scatter_peers: P->S)

The pull reads the peers' halves over NVLink and writes the destination
tensors directly, so the unpack pass of the NCCL path disappears and the
reduce-scatter sums in ascending fiber-rank order -- the reference's
`acc += b` loop (comm.py:113-125), bit for bit for every dtype.  Calls
alternate halves, so one barrier per call is enough (include/sdrng.h).

Barrier epochs come from a per-heap device counter (sdr_peer_barrier with
epoch 0), so the launches can be captured in a CUDA graph and replayed:
during capture a call that fits the existing heap records a LEADING barrier
too (every peer has then finished its pulls of earlier calls, including
replays the host never sees), and once a heap has been captured every later
eager call on it does the same.  Heap creation and regrowth cannot be
captured: warm a fiber up eagerly first, or its captured calls go to NCCL.
The graph must replay in the same stream order on every rank.

Selection (`transport()`): SDR_TRANSPORT=peer|nccl|auto (default auto = peer
when every fiber rank is on this host and its device can reach ours; the
decision is agreed by all fiber ranks).  SDR_PEER_HEAP_MB sizes the heap
(default 1024: two 512 MiB halves -- one LLaMA-3-8B layer's S->R or P->S over
a DP=2 fiber in one call); buckets larger than a half go to NCCL,
and so do collectives issued while a CUDA graph is being captured.
"""

from __future__ import annotations

import ctypes as C
import os
import socket

import torch

from . import _lib

_HEAPS: dict = {}
STATS = {"all_gather": 0, "reduce_scatter": 0, "all_reduce": 0}  # pull launches of this process
# A rank legitimately far behind its peers (checkpointing, eval, a one-time
# compile) must not trip the device barrier's trap: default to NCCL's own
# 10-minute collective timeout.
_TIMEOUT_NS = int(float(os.environ.get("SDR_PEER_TIMEOUT_S", "600")) * 1e9)


def transport() -> str:
    t = os.environ.get("SDR_TRANSPORT", "auto")
    if t not in ("auto", "peer", "nccl"):
        raise ValueError(f"SDR_TRANSPORT must be auto, peer or nccl, not {t!r}")
    return t


def _stream(dev):
    return _lib.stream_handle(dev)


class PeerHeap:
    """This rank's heap plus the mapped heaps of its fiber peers.  Created
    collectively (every fiber rank, same order) on first use of a fiber."""

    def __init__(self, group, fiber: list, dev: torch.device, half_bytes: int):
        import torch.distributed as dist
        self.dev = dev
        self.fiber = list(fiber)
        self.P = len(fiber)
        self.rank = fiber.index(dist.get_rank())
        self.half = int(half_bytes) // 256 * 256
        self.calls = 0
        self.captured = False  # a call on this heap was captured in a CUDA graph
        self.ok = False
        self._stream = None  # stream of the last call (see _order)
        self.bases: list = [None] * self.P
        total = _lib.PEER_FLAG_BYTES + 2 * self.half
        base, h = C.c_void_p(), _lib.SdrIpcHandle()
        with torch.cuda.device(dev):
            st = _lib.LIB.sdr_peer_heap_alloc(dev.index, total, C.byref(base), C.byref(h))
        _lib.check(st, "sdr_peer_heap_alloc")
        self.own = base.value
        me = (socket.gethostname(), dev.index, bytes(h.bytes))
        infos = [None] * self.P
        dist.all_gather_object(infos, me, group=group)
        reach = all(host == me[0] and (d == dev.index or torch.cuda.can_device_access_peer(dev.index, d))
                    for host, d, _ in infos)
        opened = []
        if reach:
            for q, (_, _, hb) in enumerate(infos):
                if q == self.rank:
                    self.bases[q] = self.own
                    continue
                hq = _lib.SdrIpcHandle()
                C.memmove(hq.bytes, hb, 64)
                p = C.c_void_p()
                with torch.cuda.device(dev):
                    st = _lib.LIB.sdr_peer_heap_open(dev.index, C.byref(hq), C.byref(p))
                if st != _lib.OK:
                    reach = False
                    break
                self.bases[q] = p.value
                opened.append(p.value)
        votes = [None] * self.P
        dist.all_gather_object(votes, bool(reach), group=group)
        self.ok = all(votes)
        self._flags = (C.c_void_p * self.P)(*self.bases) if self.ok else None
        if self.ok and os.environ.get("SDR_PEER_SELFCHECK", "1") != "0":
            # Known-answer check of the whole protocol (pack, barrier, reduce
            # pull, barrier, gather pull) before any user data uses it; a
            # mismatch on any rank sends the fiber to NCCL.
            good = self._self_check()
            dist.all_gather_object(votes, bool(good), group=group)
            if not all(votes):
                import warnings
                warnings.warn(f"peer transport self-check failed on fiber {fiber}: using NCCL")
                STATS["selfcheck_failed"] = STATS.get("selfcheck_failed", 0) + 1
                self.ok = False
        if not self.ok:  # give everything back: this fiber uses NCCL
            if opened:
                torch.cuda.synchronize(dev)
            for p in opened:
                _lib.LIB.sdr_peer_heap_close(p)
            dist.barrier(group=group)  # every importer closed before the owners free
            _lib.LIB.sdr_peer_heap_free(self.own)
            self.own = None
            self.bases = [None] * self.P
            self._flags = None

    def _self_check(self) -> bool:
        """All-reduce of rank-specific int32 data (ragged length, so the last
        rank's chunk is short) through this heap, compared with the sum every
        rank can compute locally.  Uses a short device-barrier timeout."""
        per = min(4099, self.half // (self.P + 1) // 4 - 8)  # fits the all-reduce's P+1 segments
        if per < 2:
            return True  # heap too small to hold a check; nothing to verify it with
        n = per * self.P - 1
        i = torch.arange(n, dtype=torch.int64, device=self.dev)
        mine = ((i * 2654435761 + 97 * self.rank) % 1000003).to(torch.int32)
        want = sum(((i * 2654435761 + 97 * q) % 1000003) for q in range(self.P)).to(torch.int32)
        out = torch.empty_like(mine)
        global _TIMEOUT_NS
        # soft barriers: a peer that never arrives sets this rank's timeout
        # word and the check fails (NCCL fallback) instead of trapping
        saved, _TIMEOUT_NS = _TIMEOUT_NS, -min(_TIMEOUT_NS, int(60e9))
        try:
            if not self.all_reduce([mine], [out]):
                return False
        finally:
            _TIMEOUT_NS = saved
        torch.cuda.synchronize(self.dev)
        STATS["all_reduce"] -= 1  # not a user collective
        word = C.c_uint64()
        with torch.cuda.device(self.dev):
            _lib.check(_lib.LIB.sdr_peer_flag_read(self.own, _lib.MAX_PEERS, C.byref(word)),
                       "sdr_peer_flag_read")
        return bool(torch.equal(out, want)) and word.value == 0

    def _order(self):
        """All work on the heap must run in call order: the one-barrier-per-call
        argument (a rank reaches barrier k+1 only after its pull of call k)
        and the monotone epochs rely on it.  Calls on one stream are ordered by
        the stream; when a call arrives on a different stream than the last
        one, it first waits for everything queued on that stream so far
        (which includes the last pull)."""
        s = torch.cuda.current_stream(self.dev)
        if torch.cuda.is_current_stream_capturing():
            # a captured call cannot wait on work outside the graph; its lead
            # barrier (_lead) orders it against every earlier pull instead
            self.captured = True
            return
        if self._stream is not None and self._stream != s:
            ev = torch.cuda.Event()
            ev.record(self._stream)
            s.wait_event(ev)
        self._stream = s

    def _half_ptrs(self, h: int):
        off = _lib.PEER_FLAG_BYTES + h * self.half
        return (C.c_void_p * self.P)(*[b + off for b in self.bases])

    def _barrier(self, stream=None):
        # epoch 0: the device counter picks it (graph-replayable)
        st = _lib.LIB.sdr_peer_barrier(self._flags, self.rank, self.P, 0, _TIMEOUT_NS,
                                       _stream(self.dev) if stream is None else stream)
        _lib.check(st, "sdr_peer_barrier")

    def _lead(self) -> int:
        """1 when this call needs a barrier before its pack: inside a CUDA
        graph capture, and on every call after one (replays are invisible to
        the host, so the half-alternation argument no longer holds)."""
        if torch.cuda.is_current_stream_capturing():
            self.captured = True
        return 1 if self.captured else 0

    def _next_half(self) -> int:
        h = self.calls & 1
        self.calls += 1
        return h

    def all_gather(self, send_members, recv_members, seg_bytes: int):
        """S->R: pack my shards into my half, barrier, pull every rank's
        segment straight into the full member tensors."""
        from .movers import CudaMover
        if seg_bytes > self.half:
            raise ValueError("bucket larger than the peer heap half")
        with torch.cuda.device(self.dev):
            self.all_gather_arrays(CudaMover._arr(send_members), CudaMover._arr(recv_members),
                                   len(send_members), _stream(self.dev))

    def all_gather_arrays(self, send_arr, recv_arr, n: int, stream: int, ordered: bool = False):
        """all_gather on prebuilt sdr_pack_member arrays (the redistribute plan
        cache patches their data pointers per call); device already current.
        One C call: pack, barrier, pull (sdr_peer_all_gather).  `ordered`:
        the caller has already run _order() for this stream."""
        if not ordered:
            self._order()
        off = _lib.PEER_FLAG_BYTES + self._next_half() * self.half
        _lib.check(_lib.LIB.sdr_peer_all_gather(send_arr, recv_arr, n, self._flags, self.P, self.rank, off,
                                                0, _TIMEOUT_NS, self._lead(), stream), "sdr_peer_all_gather")
        STATS["all_gather"] += 1

    def reduce_scatter_arrays(self, full_arr, piece_arr, n: int, seg_bytes: int, dtype_code: int,
                              stream: int, ordered: bool = False):
        """reduce_scatter on prebuilt member arrays (plan cache); device current.
        One C call: pack, barrier, reduce pull (sdr_peer_reduce_scatter)."""
        if not ordered:
            self._order()
        off = _lib.PEER_FLAG_BYTES + self._next_half() * self.half
        _lib.check(_lib.LIB.sdr_peer_reduce_scatter(full_arr, piece_arr, n, self._flags, self.P, self.rank, off,
                                                    seg_bytes, dtype_code, 0, _TIMEOUT_NS, self._lead(), stream),
                   "sdr_peer_reduce_scatter")
        STATS["reduce_scatter"] += 1

    def reduce_scatter(self, full_members, piece_members, seg_bytes: int, dtype: torch.dtype):
        """P->S: pack my Partial tensors rank-major into my half, barrier, sum
        my segment over every rank (ascending) straight into my pieces."""
        from .movers import CudaMover
        if seg_bytes * self.P > self.half:
            raise ValueError("bucket larger than the peer heap half")
        self._order()
        h = self._next_half()
        bufs = self._half_ptrs(h)
        arr = CudaMover._arr(full_members)
        with torch.cuda.device(self.dev):
            if self._lead():
                self._barrier()
            st = _lib.LIB.sdr_pack_scatter(arr, len(full_members), bufs[self.rank], seg_bytes, self.P,
                                           _stream(self.dev))
            _lib.check(st, "sdr_pack_scatter")
            self._barrier()
            arr = CudaMover._arr(piece_members)
            st = _lib.LIB.sdr_reduce_scatter_peers(arr, len(piece_members), bufs, seg_bytes, self.P,
                                                   self.rank, _SDR_DTYPE[dtype], _stream(self.dev))
        _lib.check(st, "sdr_reduce_scatter_peers")
        STATS["reduce_scatter"] += 1


    def all_reduce(self, ins: list, outs: list) -> bool:
        """P->R for contiguous tensors of one dtype: reduce-scatter pull of my
        chunk of every tensor into my half's result area, a second barrier,
        then a gather pull of every rank's reduced chunk into `outs`.  Sums
        in ascending rank order (bit-exact vs comm.py:91-101).  False (nothing
        launched) when the call does not fit a half; identical on every rank."""
        from .movers import CudaMover, Member, layout
        P = self.P
        full = [Member(t, 1, t.numel(), 1, -(-t.numel() // P)) for t in ins]
        seg = layout(full)
        if seg * (P + 1) > self.half:
            return False
        self._order()
        res = [Member(o, 1, o.numel(), 1, m.chunk, m.seg_off) for o, m in zip(outs, full)]
        h = self._next_half()
        bufs = self._half_ptrs(h)
        results = (C.c_void_p * P)(*[b + P * seg for b in bufs])
        es = ins[0].element_size()
        pieces = (_lib.SdrPackMember * max(1, len(full)))()
        for i, m in enumerate(full):
            lo = min(m.rows, self.rank * m.chunk)
            pieces[i].data = results[self.rank] + m.seg_off
            pieces[i].outer, pieces[i].inner, pieces[i].chunk_rows = 1, 1, m.chunk
            pieces[i].rows = min(m.rows, lo + m.chunk) - lo
            pieces[i].seg_off, pieces[i].elem_bytes = m.seg_off, es
        arr = CudaMover._arr(full)
        with torch.cuda.device(self.dev):
            s = _stream(self.dev)
            if self._lead():
                self._barrier()
            _lib.check(_lib.LIB.sdr_pack_scatter(arr, len(full), bufs[self.rank], seg, P, s),
                       "sdr_pack_scatter")
            self._barrier()
            _lib.check(_lib.LIB.sdr_reduce_scatter_peers(pieces, len(full), bufs, seg, P, self.rank,
                                                         _SDR_DTYPE[ins[0].dtype], s),
                       "sdr_reduce_scatter_peers")
            self._barrier()
            arr = CudaMover._arr(res)
            _lib.check(_lib.LIB.sdr_unpack_gathered_peers(arr, len(res), results, P, s),
                       "sdr_unpack_gathered_peers")
        STATS["all_reduce"] += 1
        return True


_SDR_DTYPE = {torch.float32: _lib.F32, torch.float64: _lib.F64, torch.bfloat16: _lib.BF16,
              torch.float16: _lib.F16, torch.int32: _lib.I32, torch.int64: _lib.I64}


def reducible(dtype: torch.dtype) -> bool:
    return dtype in _SDR_DTYPE


def _max_half() -> int:
    return int(float(os.environ.get("SDR_PEER_HEAP_MAX_MB", "4096")) * (1 << 20)) // 2


def heap_for(group, fiber, dev: torch.device, need_half: int = 0):
    """The fiber's PeerHeap, or None when the peer transport is off or not
    possible (then the caller uses NCCL).  Collective on first call, and when
    a call needs a larger half than the heap has (`need_half` bytes, up to
    SDR_PEER_HEAP_MAX_MB / 2): the heap is then regrown on every fiber rank
    (they all pass the same need, computed from padded segment sizes)."""
    if group is None or dev.type != "cuda" or transport() == "nccl" or len(fiber) > _lib.MAX_PEERS:
        return None
    need_half = -(-int(need_half) // 256) * 256
    key = (tuple(fiber), dev.index)
    hp = _HEAPS.get(key)
    if torch.cuda.is_current_stream_capturing():
        # a heap cannot be created or regrown inside a capture (allocation and
        # the handle exchange are not capturable): captured calls use an
        # existing heap that fits, else NCCL -- every rank captures the same
        # code with the same heaps, so all ranks agree
        return hp if hp is not None and hp.ok and need_half <= hp.half else None
    if hp is None:
        half = int(float(os.environ.get("SDR_PEER_HEAP_MB", "1024")) * (1 << 20)) // 2
        hp = _HEAPS[key] = PeerHeap(group, fiber, dev, max(half, min(need_half, _max_half())))
        if not hp.ok and transport() == "peer":
            raise RuntimeError(f"SDR_TRANSPORT=peer but fiber {fiber} cannot map peer memory")
    elif hp.ok and hp.half < need_half <= _max_half():
        hp = _HEAPS[key] = _regrow(hp, group, fiber, dev, max(need_half, 2 * hp.half))
    return hp if hp.ok else None


def _regrow(hp: PeerHeap, group, fiber, dev, half: int) -> PeerHeap:
    """Replace a fiber's heap by a larger one.  A device barrier first: every
    rank has then finished its pulls from the old halves (stream order), so
    after a host sync the mappings can be closed; a host barrier keeps the
    owners from freeing before every importer has closed."""
    import torch.distributed as dist
    with torch.cuda.device(dev):
        hp._barrier()
        torch.cuda.current_stream(dev).synchronize()
    for q, b in enumerate(hp.bases):
        if q != hp.rank and b is not None:
            _lib.LIB.sdr_peer_heap_close(b)
    dist.barrier(group=group)
    _lib.LIB.sdr_peer_heap_free(hp.own)
    STATS["regrow"] = STATS.get("regrow", 0) + 1
    return PeerHeap(group, fiber, dev, half)
