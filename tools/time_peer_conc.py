"""Whole peer-transport collectives (pack -> barrier -> pull) with P ranks
emulated as P concurrent streams of ONE GPU (tests/test_peer_gpu.py harness).
All ranks share one GPU's HBM, so the number is an HBM-side rate for the whole
pipeline (pack + barrier + pull, all ranks), not an NVLink rate:
  bytes per call = sum over ranks of (pack read+write + pull read+write).
Also: small-message latency (one 4 KiB member) per collective, device time
(all calls are enqueued behind a spin kernel before the timed interval).
"""
import ctypes as C
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import torch
from test_peer_gpu import _Ranks, _mk
from paper_2509_07003_b200 import _lib
from paper_2509_07003_b200.movers import CudaMover, layout

d, ff, kv = 4096, 14336, 1024
LAYER = [((d, d), 1), ((kv, d), 1), ((kv, d), 1), ((d, d), 0), ((ff, d), 1), ((ff, d), 1), ((d, ff), 0),
         ((d,), 0), ((d,), 0)]


def plan(P, shapes, dtype):
    rows = []
    for r in range(P):
        send, recv = [], []
        for shp, dim in shapes:
            E = shp[dim]
            c = -(-E // P)
            lo, hi = min(E, r * c), min(E, r * c + c)
            outer = int(np.prod(shp[:dim])) if dim else 1
            inner = int(np.prod(shp[dim + 1:])) if dim + 1 < len(shp) else 1
            lshape = list(shp)
            lshape[dim] = hi - lo
            send.append(_mk(torch.randn(lshape, device="cuda").to(dtype), outer, hi - lo, inner, c))
            recv.append(_mk(torch.empty(shp, device="cuda", dtype=dtype), outer, E, inner, c))
        seg = layout(send)
        for a, b in zip(send, recv):
            b.seg_off = a.seg_off
        rows.append((send, recv, seg))
    return rows


def run(R, rows, P):
    for r in range(P):
        st = R.streams[r].cuda_stream
        send, recv, seg = rows[r]
        segs = R.half_ptrs(r)
        _lib.check(_lib.LIB.sdr_pack_local(CudaMover._arr(send), len(send), segs[r], st), "pack")
        R.barrier(r)
        _lib.check(_lib.LIB.sdr_unpack_gathered_peers(CudaMover._arr(recv), len(recv), segs, P, st), "pull")


def timed(R, rows, P, reps):
    cur = torch.cuda.current_stream()
    for _ in range(3):
        run(R, rows, P)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    # hold the GPU while the host enqueues every call, so the interval is
    # device time (the one Python thread driving P ranks is not measured)
    torch.cuda._sleep(int(3e8))
    a.record(cur)
    for s in R.streams:
        s.wait_stream(cur)
    for _ in range(reps):
        run(R, rows, P)
    for s in R.streams:
        cur.wait_stream(s)
    b.record(cur)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


for P in (2, 4, 8):
    rows = plan(P, LAYER, torch.bfloat16)
    seg = rows[0][2]
    R = _Ranks(P, max(seg, 1 << 20) + (1 << 20))
    ms = timed(R, rows, P, 5)
    shard = sum(m.tensor.numel() * 2 for m in rows[0][0])
    full = sum(m.tensor.numel() * 2 for m in rows[0][1])
    per_rank = 2 * shard + 2 * full  # pack r+w, pull r+w
    small = plan(P, [((2048,), 0)], torch.bfloat16)
    lat = timed(R, small, P, 200)
    print(f"P={P} cfg5-layer S->R (all ranks on one GPU): {ms*1e3:.0f} us/call, "
          f"{P*per_rank/ms/1e6:.0f} GB/s HBM-side (pack+pull, all ranks) | "
          f"4 KiB S->R: {lat*1e3:.1f} us/call", flush=True)
    R.close()
