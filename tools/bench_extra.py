"""Secondary bench workloads (BASELINE configs 1, 3, 4, 5), same JSON shape as
bench.py's main line.  `python bench.py --workload randn|embed|init|redistribute`.

randn        cfg1: Normal(0,1) f32 [4096,4096] Shard(0) over N ranks (strong); plus the
             same window in float64 (the reference's default dtype) as a sub-object
embed        cfg3: [50257,4096] embedding on a DP x TP mesh, Shard(0),Shard(1)
             (uneven rows): Normal(0,0.02) and the std-matched Uniform, f32 and
             bf16 (strong; value = normal f32)
init         cfg4: all 291 LLaMA-3-8B params, Normal(0,0.02) bf16, TP=N (strong)
redistribute cfg5: one LLaMA-3-8B layer's params on DP x TP: fused all-gather over
             DP (S->R) then reduce-scatter of same-shaped grads (P->S); at N=1
             this measures pack + local copy + unpack only (no peers).
peer         cfg5 through the peer transport with all 8 DP2 x TP4 ranks emulated
             as concurrent streams of one GPU (tools/peer_emul.py); N=1 only.
"""
import json
import math
import os
import statistics

import numpy as np
import torch
import torch.distributed as dist

SEED = 20240817


def _env():
    return (int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
            int(os.environ.get("LOCAL_RANK", "0")))


def _time(fn, steps, warmup, dev, ws):
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize(dev)
    if ws > 1:
        dist.barrier()
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    # a short device spin queued before the start event lets the host enqueue
    # the first step while the GPU is busy, so the timed region measures the
    # steady state (a step's host work -- e.g. 3 ms to build the 291
    # descriptors of the LLaMA-3-8B init -- overlaps the previous step's GPU
    # work) instead of the first step's host latency
    torch.cuda._sleep(int(5e6))
    a.record()
    for _ in range(steps):
        fn()
    b.record()
    torch.cuda.synchronize(dev)
    if ws > 1:
        dist.barrier()
    share = os.environ.get("SDR_BENCH_SHARE_GPU") == "1"
    t = torch.tensor([a.elapsed_time(b) / steps], dtype=torch.float64, device="cpu" if share else dev)
    if ws > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.item()


_PROBE: dict = {}


def _int_roofline(per_gpu_elements_per_s: float, gpu: int) -> dict:
    """INT-roofline object of a fill line: one Philox4x32-10 block (80 INT32
    ops) per element, against the live Philox probe and
    against the IMAD.WIDE pipe ceiling (as bench.py's headline line)."""
    import ctypes as C
    from paper_2509_07003_b200 import _lib
    if gpu not in _PROBE:
        imad, lop3, phx = C.c_double(), C.c_double(), C.c_double()
        _lib.check(_lib.LIB.sdr_probe_int32(gpu, C.byref(imad), C.byref(lop3), C.byref(phx)), "sdr_probe_int32")
        _PROBE[gpu] = phx.value
    sms = torch.cuda.get_device_properties(gpu).multi_processor_count
    ceiling = sms * 32 * 1.965e9 / 20  # IMAD.WIDE blocks/s at the 1965 MHz maximum clock
    achieved = 80 * per_gpu_elements_per_s / 1e12
    return {"bound": "int32", "achieved": round(achieved, 3), "peak": round(80 * _PROBE[gpu] / 1e12, 3),
            "unit": "TOP/s INT32 (80 per Philox block, per GPU)",
            "frac": round(per_gpu_elements_per_s / _PROBE[gpu], 4),
            "pipe_ceiling": {"peak": round(80 * ceiling / 1e12, 3),
                             "frac": round(per_gpu_elements_per_s / ceiling, 4)}}


def run(a):
    from paper_2509_07003_b200 import create_mesh, init as I, rng as R
    from paper_2509_07003_b200.placement import ShardSpec, local_shape_and_offset, parse_placements
    ws, rank, local = _env()
    share = os.environ.get("SDR_BENCH_SHARE_GPU") == "1"  # test hook, as in bench.py
    gpu = 0 if share else local
    torch.cuda.set_device(gpu)
    dev = torch.device("cuda", gpu)
    if ws > 1:
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    line = {"n_gpus": ws, "steps": a.steps, "warmup": a.warmup, "higher_is_better": True,
            "vs_baseline": None, "data": "synthetic", "gpu_launches": a.steps}
    if a.workload == "randn":
        shape = (4096, 4096)
        mesh = create_mesh([("dp", ws)])
        spec = ShardSpec(mesh, parse_placements("S(0)"))
        v = local_shape_and_offset(spec, shape, mesh.coords_of_rank(rank))
        out = torch.empty(v.local_shape, dtype=torch.float32, device=dev)
        st = R.RngState(SEED)
        R.ensure_normal_tables(dev)
        ms = _time(lambda: R.fill_random(v, st, R.Normal(0, 1), np.float32, out=out), a.steps, a.warmup, dev, ws)
        n = math.prod(shape)
        line.update(metric="sharded randn GB/s (cfg1)", value=round(n * 4 / ms / 1e6, 3), unit="GB/s",
                    ms_per_step=round(ms, 4), scaling="strong", dtype="f32",
                    config={"workload": "cfg1: randn f32 [4096,4096] Shard(0)", "parallelism": f"dp{ws}",
                            "elements_per_s": round(n / ms * 1e3, 1)},
                    roofline=_int_roofline(math.prod(v.local_shape) / ms * 1e3, gpu))
        # the same window in float64, the reference's default dtype (per-point corrections)
        out64 = torch.empty(v.local_shape, dtype=torch.float64, device=dev)
        ms64 = _time(lambda: R.fill_random(v, st, R.Normal(0, 1), np.float64, out=out64), a.steps, a.warmup, dev, ws)
        line["float64"] = {"ms_per_step": round(ms64, 4), "GB/s": round(n * 8 / ms64 / 1e6, 3),
                           "elements_per_s": round(n / ms64 * 1e3, 1),
                           "int_frac": _int_roofline(math.prod(v.local_shape) / ms64 * 1e3, gpu)["frac"]}
        line["gpu_launches"] = a.steps  # (the float64 steps are a separate timed region)
    elif a.workload == "embed":
        shape = (50257, 4096)
        dp = 2 if ws % 2 == 0 else 1
        tp = ws // dp
        mesh = create_mesh([("dp", dp), ("tp", tp)])
        spec = ShardSpec(mesh, parse_placements("S(0),S(1)"))
        v = local_shape_and_offset(spec, shape, mesh.coords_of_rank(rank))
        R.ensure_normal_tables(dev)
        b = math.sqrt(3) * 0.02
        n = math.prod(shape)
        rates = {}
        for dname, dist_ in (("normal", R.Normal(0.0, 0.02)), ("uniform", R.Uniform(-b, b))):
            for dt, tdt, nm in ((np.float32, torch.float32, "f32"), ("bfloat16", torch.bfloat16, "bf16")):
                out = torch.empty(v.local_shape, dtype=tdt, device=dev)
                st = R.RngState(1234)
                ms_ = _time(lambda: R.fill_random(v, st, dist_, dt, out=out), a.steps, a.warmup, dev, ws)
                rates[f"{dname}_{nm}"] = (ms_, n * out.element_size() / ms_ / 1e6)
        ms, gbs = rates["normal_f32"]
        line.update(metric="2-D mesh embedding init GB/s (cfg3)", value=round(gbs, 3), unit="GB/s",
                    ms_per_step=round(ms, 4), scaling="strong", dtype="f32",
                    config={"workload": "cfg3: [50257,4096] S(0),S(1) on dp x tp, normal(0,0.02) f32 "
                                        "(uniform and bf16 variants in `variants`)",
                            "parallelism": f"dp{dp}xtp{tp}", "local_shape": list(v.local_shape),
                            "elements_per_s": round(n / ms * 1e3, 1),
                            "variants": {k: {"ms": round(m_, 4), "GB/s": round(g_, 1),
                                             "int_frac": _int_roofline(math.prod(v.local_shape) / m_ * 1e3, gpu)["frac"]}
                                         for k, (m_, g_) in rates.items()}},
                    roofline=_int_roofline(math.prod(v.local_shape) / ms * 1e3, gpu))
    elif a.workload == "init":
        params = I.llama3_8b_params(lambda nm, s: R.Normal(0.0, 0.02), "bfloat16")
        mesh = create_mesh([("tp", ws)])
        specs = I.llama3_tp_specs(params, mesh)
        coord = mesh.coords_of_rank(rank)
        n_local = sum(math.prod(local_shape_and_offset(specs[k], p.shape, coord).local_shape)
                      for k, p in params.items())
        total = sum(math.prod(p.shape) for p in params.values())

        def step():
            for p in params.values():
                p.value = None
            I.materialize(params, R.RngState(SEED), specs, coord, device=dev)
        ms = _time(step, a.steps, a.warmup, dev, ws)
        # unique elements across ranks (norms are replicated: count once)
        line.update(metric="LLaMA-3-8B sharded init GB/s (cfg4)", value=round(total * 2 / ms / 1e6, 3),
                    unit="GB/s", ms_per_step=round(ms, 3), scaling="strong", dtype="bf16",
                    config={"workload": "cfg4: LLaMA-3-8B 291 params normal(0,0.02) bf16, TP placements",
                            "parallelism": f"tp{ws}", "per_gpu_elements": n_local,
                            "elements_per_s": round(total / ms * 1e3, 1)},
                    roofline=_int_roofline(n_local / ms * 1e3, gpu))
    elif a.workload == "peer":
        if ws > 1:
            raise SystemExit("--workload peer emulates all cfg5 ranks on one GPU: run it with N=1")
        from tools.peer_emul import Emulated
        em = Emulated()
        cur = torch.cuda.current_stream(dev)
        for _ in range(a.warmup):
            em.step()
        ok = em.check()
        torch.cuda.synchronize(dev)
        ev0, ev1 = torch.cuda.Event(True), torch.cuda.Event(True)
        torch.cuda._sleep(int(4e8))  # the host enqueues all steps of all 8 streams behind this
        ev0.record(cur)
        for s_ in em.streams:
            s_.wait_stream(cur)
        for _ in range(a.steps):
            em.step()
        for s_ in em.streams:
            cur.wait_stream(s_)
        ev1.record(cur)
        torch.cuda.synchronize(dev)
        ms = ev0.elapsed_time(ev1) / a.steps
        nbytes = em.hbm_bytes_per_step()
        em.close()
        try:
            with open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                   "MEASURED_PEAKS.json")) as f:
                hbm_peak = float(json.load(f)["hbm_gbs"])
        except (OSError, KeyError, ValueError):
            hbm_peak = 6650.0  # fallback figure of B200_PROFILING.md
        gbs = nbytes / ms / 1e6
        line.update(metric="cfg5 fused redistribute via peer transport, all 8 ranks emulated on one GPU "
                           "(HBM-side GB/s)", value=round(gbs, 1), unit="GB/s", ms_per_step=round(ms, 4),
                    scaling="none", dtype="bf16", gpu_launches=a.steps * em.n * 6,
                    roofline={"bound": "hbm", "achieved": round(gbs, 1), "peak": hbm_peak, "unit": "GB/s",
                              "frac": round(gbs / hbm_peak, 4), "traffic": None},
                    config={"workload": "cfg5: one LLaMA-3-8B layer on DP2 x TP4; per step every rank "
                                        "does the fused S->R all-gather over its DP fiber and the fused "
                                        "P->S reduce-scatter of same-shaped grads (pack -> device barrier "
                                        "-> pull kernel), 8 ranks as 8 concurrent streams of one GPU",
                            "parallelism": "dp2xtp4 emulated", "bit_exact_check": ok,
                            "hbm_bytes_per_step": nbytes,
                            "note": "all ranks share one GPU's HBM: this is the pipeline's HBM-side rate, "
                                    "not an NVLink rate"})
    else:
        from paper_2509_07003_b200 import peer
        from paper_2509_07003_b200.dtensor import from_local, redistribute_many
        dp = 2 if ws % 2 == 0 else 1
        tp = ws // dp
        mesh = create_mesh([("dp", dp), ("tp", tp)])
        coord = mesh.coords_of_rank(rank)
        d, ff, kv = 4096, 14336, 1024
        layer = {"q": ((d, d), "S(1),S(0)"), "k": ((kv, d), "S(1),S(0)"), "v": ((kv, d), "S(1),S(0)"),
                 "o": ((d, d), "S(0),S(1)"), "gate": ((ff, d), "S(1),S(0)"), "up": ((ff, d), "S(1),S(0)"),
                 "down": ((d, ff), "S(0),S(1)"), "n1": ((d,), "S(0),R"), "n2": ((d,), "S(0),R")}
        xs, dsts, grads, gdst = [], [], [], []
        for name, (shape, pl) in layer.items():
            spec = ShardSpec(mesh, parse_placements(pl))
            v = local_shape_and_offset(spec, shape, coord)
            xs.append(from_local(torch.randn(v.local_shape, device=dev, dtype=torch.bfloat16), spec, shape, coord))
            dst_pl = ["R"] + [str(p) for p in spec.placements[1:]]
            dsts.append(ShardSpec(mesh, parse_placements(",".join(dst_pl))))
            gspec = ShardSpec(mesh, parse_placements(",".join(["P"] + dst_pl[1:])))
            gv = local_shape_and_offset(gspec, shape, coord)
            grads.append(from_local(torch.randn(gv.local_shape, device=dev, dtype=torch.bfloat16), gspec, shape, coord))
            gdst.append(spec)
        ms_ag = _time(lambda: redistribute_many(xs, dsts), a.steps, a.warmup, dev, ws)
        ms_rs = _time(lambda: redistribute_many(grads, gdst), a.steps, a.warmup, dev, ws)
        S = sum(math.prod(x.shape) // tp for x in xs) * 2  # gathered bytes per DP fiber
        if dp > 1:
            busbw = lambda ms: S / ms / 1e6 * (dp - 1) / dp
            metric = "fused redistribute busBW (cfg5)"
        else:  # one-rank DP fiber: no exchange; report the local data movement (read + write)
            busbw = lambda ms: 2 * S / ms / 1e6
            metric = "fused redistribute local copy GB/s (cfg5 at dp=1: no exchange)"
        line.update(metric=metric, value=round(busbw(ms_ag), 3), unit="GB/s",
                    ms_per_step=round(ms_ag, 4), scaling="weak", dtype="bf16",
                    config={"workload": "cfg5: one LLaMA-3-8B layer, fused AG (S->R over dp) + RS (P->S)",
                            "parallelism": f"dp{dp}xtp{tp}", "ms_allgather": round(ms_ag, 4),
                            "ms_reducescatter": round(ms_rs, 4),
                            "busbw_reducescatter": round(busbw(ms_rs), 3),
                            "payload_bytes_per_fiber": S,
                            # peer-memory pulls (peer.py) or NCCL; SDR_TRANSPORT=nccl forces NCCL
                            "transport": "peer" if peer.STATS["all_gather"] else
                                         ("nccl" if dp > 1 else "none")})
    if rank == 0:
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()


# ---------------------------------------------------------------------------
# cfg5 summary for the headline line at WORLD_SIZE > 1 (bench.py).
# ---------------------------------------------------------------------------
def cfg5_redistribute(steps: int, warmup: int, dev, ws: int, rank: int, share: bool) -> dict:
    """One LLaMA-3-8B layer's 9 params on a DP x TP mesh (DP = 2): the fused
    S->R all-gather over DP (`redistribute_many`) and the fused P->S
    reduce-scatter of same-shaped grads, each through the peer transport and
    through NCCL, against per-tensor `redistribute` calls and ONE
    single-buffer NCCL collective of the same bytes (the busBW ceiling of the
    >= 80% target).  busBW = S (P-1)/P / t, S = gathered bytes per DP fiber
    (NCCL-tests convention = the reference ledger's, comm.py:45-62).  Values:
    params Uniform(-1,1) and integer-valued grads (RandInt, so any summation
    order is exact) drawn from the parity-tested RNG by global index, so every
    expected output is computable on each rank: `bit_exact` compares every
    measured variant's outputs with it, bit for bit."""
    import math
    from paper_2509_07003_b200 import create_mesh, peer, rng as R
    from paper_2509_07003_b200 import dtensor as DT
    from paper_2509_07003_b200.comm import fiber_group
    from paper_2509_07003_b200.placement import ShardSpec, local_shape_and_offset, parse_placements
    if ws % 2:
        return {"skipped": "odd world size: no DP=2 fiber"}
    dp, tp = 2, ws // 2
    mesh = create_mesh([("dp", dp), ("tp", tp)])
    coord = mesh.coords_of_rank(rank)
    d, ff, kv = 4096, 14336, 1024
    layer = {"q": ((d, d), "S(1),S(0)"), "k": ((kv, d), "S(1),S(0)"), "v": ((kv, d), "S(1),S(0)"),
             "o": ((d, d), "S(0),S(1)"), "gate": ((ff, d), "S(1),S(0)"), "up": ((ff, d), "S(1),S(0)"),
             "down": ((d, ff), "S(0),S(1)"), "n1": ((d,), "S(0),R"), "n2": ((d,), "S(0),R")}
    xs, dsts, grads, gdst, exp_ag, exp_rs = [], [], [], [], [], []
    for i, (name, (shape, pl)) in enumerate(layer.items()):
        spec = ShardSpec(mesh, parse_placements(pl))
        dst_pl = ["R"] + [str(p) for p in spec.placements[1:]]
        dspec = ShardSpec(mesh, parse_placements(",".join(dst_pl)))
        gspec = ShardSpec(mesh, parse_placements(",".join(["P"] + dst_pl[1:])))
        st = R.RngState(1000 + i)
        u = R.Uniform(-1.0, 1.0)
        xs.append(DT.from_local(R.fill_random(local_shape_and_offset(spec, shape, coord), st, u, "bfloat16",
                                              device=dev), spec, shape, coord))
        dsts.append(dspec)
        exp_ag.append(R.fill_random(local_shape_and_offset(dspec, shape, coord), st, u, "bfloat16", device=dev))
        # rank-dependent Partial grads: dp index k draws with seed 2000 + 16 i + k
        ri = R.RandInt(-8, 8)
        gv = local_shape_and_offset(gspec, shape, coord)
        g = R.fill_random(gv, R.RngState(2000 + 16 * i + coord[0]), ri, np.float32, device=dev)
        grads.append(DT.from_local(g.to(torch.bfloat16), gspec, shape, coord))
        gdst.append(spec)
        pv = local_shape_and_offset(spec, shape, coord)
        acc = sum(R.fill_random(pv, R.RngState(2000 + 16 * i + k), ri, np.float32, device=dev)
                  for k in range(dp))
        exp_rs.append(acc.to(torch.bfloat16))
    S = sum(x.numel() * 2 for x in exp_ag)  # gathered bytes per rank (= per DP fiber member)
    busbw = lambda ms: round(S / ms / 1e6 * (dp - 1) / dp, 2)

    def same(outs, exp):
        return all(torch.equal(o.to_local().view(torch.int16), e.view(torch.int16)) for o, e in zip(outs, exp))

    env0 = {k: os.environ.get(k) for k in ("SDR_TRANSPORT", "SDR_COMM_CPU_STAGING")}
    res, exact = {}, {}
    try:
        for tname in ("peer", "nccl"):
            os.environ["SDR_TRANSPORT"] = tname
            if share and tname == "nccl":
                os.environ["SDR_COMM_CPU_STAGING"] = "1"  # gloo stand-in: NCCL refuses 2 ranks on 1 GPU
            n0 = dict(peer.STATS)
            ag = DT.redistribute_many(xs, dsts)
            rs = DT.redistribute_many(grads, gdst)
            torch.cuda.synchronize(dev)
            exact[f"fused_{tname}"] = bool(same(ag, exp_ag) and same(rs, exp_rs))
            used_peer = peer.STATS["all_gather"] > n0["all_gather"]
            if tname == "peer" and not used_peer:
                res["fused_peer"] = {"unavailable": "peer memory not reachable on this fiber"}
                continue
            ms_ag = _time(lambda: DT.redistribute_many(xs, dsts), steps, warmup, dev, ws)
            ms_rs = _time(lambda: DT.redistribute_many(grads, gdst), steps, warmup, dev, ws)
            res[f"fused_{tname}"] = {"ag_ms": round(ms_ag, 4), "ag_busbw": busbw(ms_ag),
                                     "rs_ms": round(ms_rs, 4), "rs_busbw": busbw(ms_rs),
                                     **({"via": "gloo host staging (ranks share one GPU)"}
                                        if share and tname == "nccl" else {})}
        # per-tensor redistribute calls over NCCL (9 collectives per direction)
        os.environ["SDR_TRANSPORT"] = "nccl"
        ag1 = [DT.redistribute(x, dd) for x, dd in zip(xs, dsts)]
        rs1 = [DT.redistribute(g, dd) for g, dd in zip(grads, gdst)]
        torch.cuda.synchronize(dev)
        exact["per_tensor_nccl"] = bool(same(ag1, exp_ag) and same(rs1, exp_rs))
        ms_ag = _time(lambda: [DT.redistribute(x, dd) for x, dd in zip(xs, dsts)], steps, warmup, dev, ws)
        ms_rs = _time(lambda: [DT.redistribute(g, dd) for g, dd in zip(grads, gdst)], steps, warmup, dev, ws)
        res["per_tensor_nccl"] = {"ag_ms": round(ms_ag, 4), "ag_busbw": busbw(ms_ag),
                                  "rs_ms": round(ms_rs, 4), "rs_busbw": busbw(ms_rs)}
        # one single-buffer collective of the same bytes on the DP fiber group
        if share:
            res["single_buffer_nccl"] = {"unavailable": "ranks share one GPU (NCCL: duplicate GPU)"}
        else:
            group, _ = fiber_group(mesh, (0,))
            send = torch.empty(S // dp // 2, dtype=torch.bfloat16, device=dev)
            recv = torch.empty(S // 2, dtype=torch.bfloat16, device=dev)
            ms_ag = _time(lambda: dist.all_gather_into_tensor(recv, send, group=group), steps, warmup, dev, ws)
            ms_rs = _time(lambda: dist.reduce_scatter_tensor(send, recv, group=group), steps, warmup, dev, ws)
            res["single_buffer_nccl"] = {"ag_ms": round(ms_ag, 4), "ag_busbw": busbw(ms_ag),
                                         "rs_ms": round(ms_rs, 4), "rs_busbw": busbw(ms_rs)}
    finally:
        for k, v in env0.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    out = {"workload": "cfg5: one LLaMA-3-8B layer (9 params), fused S->R all-gather over DP and P->S "
                       "reduce-scatter of same-shaped grads", "mesh": f"dp{dp}xtp{tp}",
           "gathered_bytes_per_rank": S, "unit": "GB/s busBW (S (P-1)/P / t)", **res,
           "bit_exact": exact, "steps": steps}
    ceil = res.get("single_buffer_nccl", {})
    for tname in ("fused_peer", "fused_nccl"):
        r = res.get(tname, {})
        if "ag_busbw" in r and "ag_busbw" in ceil:
            r["ag_frac_of_single_buffer"] = round(r["ag_busbw"] / ceil["ag_busbw"], 3)
            r["rs_frac_of_single_buffer"] = round(r["rs_busbw"] / ceil["rs_busbw"], 3)
    return out
