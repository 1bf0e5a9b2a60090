"""Benchmark: sharded dropout (BASELINE config 2) on 1..N B200s.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...      (N > 1)

Workload (BASELINE.json configs[1]): x = bf16 [8, 4096, 4096] activations
(synthetic, torch.randn seed 0), dropout p = 0.1, Shard(1) (sequence parallel)
over the N ranks of a 1-d mesh.  The global tensor is fixed, so scaling is
strong: rank r owns x[:, r*4096/N : (r+1)*4096/N, :].

A step = one forward dropout of the rank's shard with single-device semantics:
the keep-mask is the rank's slice of ONE global Bernoulli(0.9) draw from the
shared RngState (no communication), y = (x*m)*(1/0.9) in one fused sm_100a
kernel (mask not stored; backward regenerates it).  Metric: GB/s of
algorithmic bytes (read x 2 B + write y 2 B per element), whole job.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

SHAPE = (8, 4096, 4096)
P_DROP = 0.1
SEED = 20240817
METRIC = "sharded randn/dropout GB/s per GPU & aggregate at 1/2/4/8 B200 vs roofline; bit-exact"
BYTES_PER_ELEM = 4  # bf16 read + bf16 write
PHILOX_OPS = 80     # INT32 ops per Philox4x32-10 block


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--workload", choices=["dropout", "randn", "embed", "init", "redistribute", "peer"],
                    default="dropout",
                    help="dropout = BASELINE cfg2 (the driver's line); the others are the secondary "
                         "configs 1, 3, 4 and 5, printed in the same JSON shape")
    return ap.parse_args()


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


# ---------------------------------------------------------------------------
# CPU side: the oracle port of the reference path, timed on host cores.
# ---------------------------------------------------------------------------
def _cpu_sample(args):
    """Dropout of rows [r0, r0+nrows) of batch b: mask via the oracle's
    restatement of rng.py + engine.k_dropout_apply (numpy, 1 core)."""
    import ml_dtypes
    import numpy as np
    from oracle import rng_oracle as O
    b, r0, nrows, seed = args
    rs = np.random.default_rng(b * 100003 + r0)
    x = rs.standard_normal((nrows, SHAPE[2]), dtype=np.float32).astype(ml_dtypes.bfloat16)
    j = (np.arange(nrows * SHAPE[2], dtype=np.int64) + (b * SHAPE[1] + r0) * SHAPE[2])
    t0 = time.perf_counter()
    keep = O.fill_indices(j, seed, 0, 65536, "bernoulli", (1.0 - P_DROP,), ml_dtypes.bfloat16)
    y = O.dropout_apply(x.reshape(-1), keep, P_DROP)
    dt = time.perf_counter() - t0
    return dt, y.size


def cpu_measure(n_elems: int, cores: int, piece_rows: int = 2048):
    """Time the oracle on `n_elems` elements split over `cores` processes
    (each process works through pieces of at most `piece_rows` rows to bound
    its memory).  The rate counts compute time only -- the slowest process's
    sum of per-piece times, not data generation or pool start-up -- so the
    CPU number is the most favourable one.  Returns (elements/s, seconds, elements)."""
    rows = max(1, n_elems // SHAPE[2])
    per = max(1, rows // cores)
    jobs = []
    for i in range(cores):
        for r0 in range(0, per, piece_rows):
            jobs.append((i, (0, i * per + r0, min(piece_rows, per - r0), SEED)))
    if cores == 1:
        res = [(0, _cpu_sample(j)) for _, j in jobs]
    else:
        import multiprocessing as mp
        with mp.get_context("fork").Pool(cores) as pool:
            out = pool.map(_cpu_sample, [j for _, j in jobs])
        res = list(zip([w for w, _ in jobs], out))
    busy = {}
    for w, (dt, _) in res:
        busy[w] = busy.get(w, 0.0) + dt
    secs = max(busy.values())
    elems = sum(n for _, (_, n) in res)
    return elems / secs, secs, elems


def cpu_info() -> dict:
    """Host CPU model, usable cores and NumPy's SIMD dispatch (BASELINE.md
    section 2 asks for them next to every CPU number)."""
    import numpy as np
    model = ""
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    model = ln.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    simd = {}
    try:
        from numpy._core._multiarray_umath import __cpu_baseline__, __cpu_dispatch__, __cpu_features__
        simd = {"baseline": list(__cpu_baseline__),
                "dispatch_found": [f for f in __cpu_dispatch__ if __cpu_features__.get(f)]}
    except ImportError:
        pass
    return {"cpu_model": model, "nproc": os.cpu_count(),
            "affinity": len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else None,
            "numpy": np.__version__, "numpy_simd": simd}


def parity_check(y, x, view, seed: int, offset: int, n_rows: int = 256) -> dict:
    """Checker for the timed output: `n_rows` rows of 4096 elements spread over
    this rank's shard (every batch, sequence positions spread across the shard)
    of the LAST timed step's y, against the oracle restatement of
    rng.py:185-242 + engine.py:80-81 (the reference's f32 result, rounded to
    bf16).  The oracle is only the checker here."""
    import ml_dtypes
    import numpy as np
    import torch
    from oracle import rng_oracle as O
    B, n, W = view.local_shape
    s0 = view.local_offset[1]
    per_b = max(1, n_rows // B)
    rows = [(b, int(s)) for b in range(B) for s in np.linspace(0, n - 1, min(per_b, n)).round()]
    bi = torch.tensor([r[0] for r in rows], device=y.device)
    si = torch.tensor([r[1] for r in rows], device=y.device)
    ys = y[bi, si].cpu().view(torch.int16).numpy().view(np.uint16)
    xs = x[bi, si].cpu().view(torch.int16).numpy().view(np.uint16).view(ml_dtypes.bfloat16)
    rb = np.array([r[0] for r in rows], dtype=np.int64)
    rs = np.array([r[1] for r in rows], dtype=np.int64)
    j = (((rb * SHAPE[1] + s0 + rs) * SHAPE[2])[:, None] + np.arange(W, dtype=np.int64)[None, :]).reshape(-1)
    keep = O.fill_indices(j, seed, offset, 65536, "bernoulli", (1.0 - P_DROP,), ml_dtypes.bfloat16)
    ref = O.dropout_apply(xs.reshape(-1), keep, P_DROP).astype(ml_dtypes.bfloat16).view(np.uint16)
    bad = int(np.count_nonzero(ref != ys.reshape(-1)))
    return {"checked": int(ref.size), "mismatches": bad,
            "what": f"{len(rows)} rows x {W} of the last timed step's y (all batches, sequence rows "
                    f"spread over the shard) vs oracle/rng_oracle.py (rng.py:185-242 + engine.py:80-81) "
                    f"rounded to bf16"}


def run_reference(a):
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    cores = os.cpu_count() or 1
    sample = 2 * cores * SHAPE[2] * 64  # 64 rows per core per step
    for _ in range(a.warmup):
        cpu_measure(sample // 8, cores)
    rates, walls = [], []
    for _ in range(a.steps):
        r, wall, _ = cpu_measure(sample, cores)
        rates.append(r)
        walls.append(wall)
    rate = statistics.median(rates)
    gbs = rate * BYTES_PER_ELEM / 1e9
    ms = statistics.median(walls) * 1e3  # one bounded-sample step
    line = {
        "impl": "reference", "metric": METRIC, "value": round(gbs, 6), "unit": "GB/s",
        "n_gpus": ws, "steps": a.steps, "warmup": a.warmup, "ms_per_step": round(ms, 3),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic",
        "config": {"workload": "cfg2: dropout p=0.1 on bf16 [8,4096,4096], Shard(1) sequence-parallel",
                   "global_shape": list(SHAPE), "p": P_DROP, "placement": "S(1)",
                   "parallelism": f"sp{ws}"},
        "cpu_baseline": {"value": round(gbs, 6), "unit": "GB/s", "cores": cores, "kind": "port",
                         "sample": f"{sample} elements per step ({cores} procs x 64 rows x 2 x 4096),"
                                   " numpy restatement of rng.py + engine.k_dropout_apply",
                         "host": cpu_info()},
        "e2e": {"value": round(gbs, 6), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# GPU side.
# ---------------------------------------------------------------------------
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.gpu = gpu_index
        self.p = None

    def __enter__(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "100"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except OSError:
            self.p = None
        time.sleep(0.25)
        return self

    def __exit__(self, *exc):
        if self.p is not None:
            self.p.terminate()
            self.p.wait()
        return False

    def summary(self):
        self.f.flush()
        self.f.seek(0)
        sm, mx, reasons = [], 0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.f.read().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx = max(mx, float(parts[2]))
            except ValueError:
                continue
            for n, v in zip(names, parts[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def run_ours(a):
    import numpy as np
    import torch
    import torch.distributed as dist

    ws, rank, local = dist_env()
    if ws != a.gpus:
        raise SystemExit(f"--gpus {a.gpus} but WORLD_SIZE={ws}")
    # Test hook: SDR_BENCH_SHARE_GPU=1 runs every rank on cuda:0 with gloo for the
    # barriers / max-over-ranks (exercises the N-rank path on a 1-GPU box; the
    # numbers are then not scaling numbers).
    share = os.environ.get("SDR_BENCH_SHARE_GPU") == "1"
    gpu = 0 if share else local
    torch.cuda.set_device(gpu)
    dev = torch.device("cuda", gpu)
    if ws > 1:
        if share:
            dist.init_process_group("gloo")
        else:
            # communicator init lines (rank / nRanks per comm) on stderr
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            dist.init_process_group("nccl", device_id=dev)

    from paper_2509_07003_b200 import _lib, create_mesh, ops, rng as R
    from paper_2509_07003_b200.placement import ShardSpec, local_shape_and_offset, parse_placements

    mesh = create_mesh([("sp", ws)])
    spec = ShardSpec(mesh, parse_placements("S(1)"))
    view = local_shape_and_offset(spec, SHAPE, mesh.coords_of_rank(rank))
    s0, n = view.local_offset[1], view.local_shape[1]
    gen = torch.Generator(device=dev).manual_seed(0)
    x_full_rows = torch.randn((SHAPE[0], SHAPE[1], SHAPE[2]), generator=gen, device=dev,
                              dtype=torch.bfloat16) if ws == 1 else None
    if ws == 1:
        x = x_full_rows
    else:  # same synthetic global tensor, generated per batch to bound memory
        x = torch.empty(view.local_shape, dtype=torch.bfloat16, device=dev)
        for b in range(SHAPE[0]):
            xb = torch.randn((SHAPE[1], SHAPE[2]), generator=gen, device=dev, dtype=torch.bfloat16)
            x[b].copy_(xb[s0:s0 + n])
            del xb
    n_local = x.numel()
    local_bytes = n_local * BYTES_PER_ELEM
    # Rotate over enough (x, y) buffer pairs that the footprint exceeds 3x L2:
    # every step reads an x that is not L2-resident (no flush kernel needed),
    # and the K steps run back to back between one pair of events.
    l2_bytes = 126 * 1024 * 1024
    nbuf = max(1, math.ceil(3 * l2_bytes / local_bytes))  # local_bytes = x + y bytes
    xs = [x] + [x.clone() for _ in range(nbuf - 1)]
    ys = [torch.empty_like(x) for _ in range(nbuf)]
    stream = torch.cuda.current_stream(dev)
    state = R.RngState(SEED, 0, 65536)

    last = {}

    def step(i):
        last["i"], last["offset"] = i, state.offset  # which buffer / offset the parity check reads
        ops.dropout_apply(xs[i % nbuf], P_DROP, state, view, out=ys[i % nbuf])
        state.advance(math.prod(SHAPE))  # every rank, no communication (rng.py:95-98)

    for i in range(a.warmup):
        step(i)
    torch.cuda.synchronize(dev)

    # --- timed region: K steps, barrier + synchronize on both sides ---------
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    with ClockSampler(gpu) as clk:
        # Keep the GPU under this same load for ~0.4 s before the timed steps so
        # the 100 ms nvidia-smi samples see the clocks of the workload (the K
        # timed steps alone last only a few ms); these extra steps are untimed.
        # (the state is not advanced here, so every rank's offset stays identical)
        spin, t_spin = 0, time.perf_counter()
        while time.perf_counter() - t_spin < 0.4:
            for _ in range(8):
                ops.dropout_apply(xs[spin % nbuf], P_DROP, state, view, out=ys[spin % nbuf])
                spin += 1
            torch.cuda.synchronize(dev)
        if ws > 1:
            dist.barrier()
        t0.record(stream)
        for i in range(a.steps):
            step(i)
        t1.record(stream)
        torch.cuda.synchronize(dev)
        if ws > 1:
            dist.barrier()
    ms_local = t0.elapsed_time(t1) / a.steps
    clocks = clk.summary()
    # parity of the last timed step's output (every rank checks its own shard)
    par = parity_check(ys[last["i"] % nbuf], xs[last["i"] % nbuf], view, SEED, last["offset"])

    # --- e2e through the public API with host buffers -------------------------
    # Every step copies its input x from pinned host memory to the GPU and its
    # result y back to pinned host memory (ops.dropout_host).  Steps are issued
    # stream-ordered without a host sync in between (sync=False, two host
    # output buffers in rotation), like a prefetching input pipeline, so PCIe
    # stays busy in both directions across steps; one event pair brackets the
    # K steps and the host synchronizes at the end.  The per-step-synchronous
    # rate is reported beside it.
    xh = x.cpu().pin_memory()
    yhs = [torch.empty_like(xh).pin_memory() for _ in range(2)]
    st2 = R.RngState(SEED, 0, 65536)

    def e2e_step(i, sync):
        ops.dropout_host(xh, P_DROP, st2, view, out=yhs[i % 2], device=dev, sync=sync)
        st2.advance(math.prod(SHAPE))

    for i in range(2):
        e2e_step(i, True)
    torch.cuda.synchronize(dev)
    if ws > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for i in range(a.steps):
        e2e_step(i, False)
    e1.record(stream)
    torch.cuda.synchronize(dev)
    e2e_ms_local = e0.elapsed_time(e1) / a.steps
    if ws > 1:
        dist.barrier()
    e0.record(stream)
    for i in range(a.steps):
        e2e_step(i, True)
    e1.record(stream)
    torch.cuda.synchronize(dev)
    e2e_sync_ms_local = e0.elapsed_time(e1) / a.steps
    yh = yhs[0]

    # --- max over ranks -------------------------------------------------------
    t = torch.tensor([ms_local, e2e_ms_local, e2e_sync_ms_local], dtype=torch.float64,
                     device="cpu" if share else dev)
    if ws > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms, e2e_ms, e2e_sync_ms = t.tolist()
    pt = torch.tensor([par["checked"], par["mismatches"]], dtype=torch.int64,
                      device="cpu" if share else dev)
    if ws > 1:
        dist.all_reduce(pt, op=dist.ReduceOp.SUM)
    par["checked"], par["mismatches"] = (int(v) for v in pt.tolist())
    par["ranks"] = ws
    total_elems = math.prod(SHAPE)
    gbs = total_elems * BYTES_PER_ELEM / (ms * 1e-3) / 1e9
    e2e_gbs = total_elems * BYTES_PER_ELEM / (e2e_ms * 1e-3) / 1e9
    e2e_sync_gbs = total_elems * BYTES_PER_ELEM / (e2e_sync_ms * 1e-3) / 1e9

    # --- roofline (rank 0's kernel) --------------------------------------------
    peaks = {}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            peaks = json.load(f)
    except OSError:
        pass
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    hbm_src = "MEASURED_PEAKS.json" if "hbm_gbs" in peaks else "fallback B200_PROFILING.md"
    import ctypes as C
    imad, lop3, phx = C.c_double(), C.c_double(), C.c_double()
    _lib.check(_lib.LIB.sdr_probe_int32(gpu, C.byref(imad), C.byref(lop3), C.byref(phx)),
               "sdr_probe_int32")
    # INT32 peak in Philox proportion: a memory-free Philox4x32-10 with every
    # counter word per-thread varying and all four words consumed (nothing to
    # hoist), x 80 INT32 ops per block.
    int_peak_tops = PHILOX_OPS * phx.value / 1e12
    # Issue ceiling of the fma-heavy pipe: IMAD.WIDE.U32 issues at 32 per SM per
    # clock (4 cycles per warp per SMSP), a Philox block is
    # 20 of them -> SMs x 32 x f_max / 20 blocks/s.
    sm_max_hz = (clocks.get("sm_max_mhz") or 1965.0) * 1e6
    n_sms = torch.cuda.get_device_properties(dev).multi_processor_count
    ceil_blocks = n_sms * 32 * sm_max_hz / 20
    ceil_tops = PHILOX_OPS * ceil_blocks / 1e12
    achieved_tops = n_local / (ms_local * 1e-3) * PHILOX_OPS / 1e12
    achieved_gbs_local = local_bytes / (ms_local * 1e-3) / 1e9

    traffic = None
    try:  # dram bytes of this kernel from the committed ncu capture (profiles/)
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            tr = json.load(f)["k_dropout_fast"]
        traffic = (tr["dram_bytes_read"] + tr["dram_bytes_write"]) * (n_local / math.prod(SHAPE))
    except (OSError, KeyError, ValueError):
        pass

    line = None
    if rank == 0:
        cpu = None
        if not a.no_cpu_baseline and ws == 1:
            sample = 12 * 1024 * SHAPE[2]  # 50 M elements, 1 core, ~15 s of compute
            rate, secs, elems = cpu_measure(sample, 1)
            cpu = {"value": round(rate * BYTES_PER_ELEM / 1e9, 6), "unit": "GB/s", "cores": 1,
                   "kind": "port", "host": cpu_info(),
                   "sample": f"{elems} elements (rows 0-12287 x 4096 of batch 0, 6 pieces), numpy "
                             f"restatement of rng.py:185-242 + engine.py:80-81, {secs:.1f}s of compute"}
        line = {
            "metric": METRIC, "value": round(gbs, 3), "unit": "GB/s", "n_gpus": ws,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": round(ms, 4),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic",
            "config": {"workload": "cfg2: dropout p=0.1 on bf16 [8,4096,4096], Shard(1) sequence-parallel",
                       "global_shape": list(SHAPE), "p": P_DROP, "placement": "S(1)",
                       "parallelism": f"sp{ws}", "per_gpu_elements": n_local,
                       "l2": f"{nbuf} rotating x/y buffer pair(s), {nbuf * local_bytes // 2**20} MiB "
                             f"footprint > 3x the 126 MB L2 (no step reads an L2-resident x)",
                       "timing": "one CUDA-event pair around the K back-to-back steps on the launch stream",
                       "per_gpu_gbs": round(gbs / ws, 3),
                       "elements_per_s": round(total_elems / (ms * 1e-3), 1)},
            "roofline": {
                "bound": "int32", "achieved": round(achieved_tops, 3), "peak": round(int_peak_tops, 3),
                "unit": "TOP/s INT32 (80 per Philox block)", "frac": round(achieved_tops / int_peak_tops, 4),
                "traffic": traffic, "traffic_note": "dram read+write bytes per launch, ncu (profiles/traffic.json); "
                                                    "algorithmic bytes per launch = %d" % local_bytes,
                "int32_probe": {"imad_wide_per_s": imad.value, "lop3_per_s": lop3.value,
                                "philox_blocks_per_s_no_hoist": phx.value,
                                "how": "sdr_probe_int32 live: peak = 80 x philox_blocks_per_s_no_hoist; "
                                       "imad_wide/lop3 = independent non-foldable chains (probe.cu)"},
                "pipe_ceiling": {"peak": round(ceil_tops, 3), "frac": round(achieved_tops / ceil_tops, 4),
                                 "how": f"{n_sms} SMs x 32 IMAD.WIDE/clk x {sm_max_hz / 1e6:.0f} MHz / "
                                        "20 per block x 80 ops"},
                "hbm": {"achieved": round(achieved_gbs_local, 1), "peak": hbm_peak, "unit": "GB/s",
                        "frac": round(achieved_gbs_local / hbm_peak, 4), "peak_source": hbm_src},
                "kernel": "k_dropout_fast<BF16,BF16,-1> (one launch per step)",
            },
            "e2e": {"value": round(e2e_gbs, 3), "unit": "GB/s",
                    "h2d_bytes_per_step": xh.numel() * xh.element_size(),
                    "d2h_bytes_per_step": yh.numel() * yh.element_size(),
                    "sync_per_step_value": round(e2e_sync_gbs, 3),
                    "how": "paper_2509_07003_b200.ops.dropout_host: pinned host x -> H2D | fused kernel | "
                           "D2H y (tapered 3-stream block pipeline); K steps issued stream-ordered "
                           "(sync=False), one host sync at the end; sync_per_step_value = host sync "
                           "after every step"},
            "gpu_launches": a.steps,
            "clocks": clocks,
            "parity": par,
        }
        if cpu is not None:
            line["cpu_baseline"] = cpu
    if ws > 1:
        # second north-star target: cfg5 fused redistribute busBW (after the headline timing)
        from tools.bench_extra import cfg5_redistribute
        red = cfg5_redistribute(10, 3, dev, ws, rank, share)
        if rank == 0:
            line["redistribute"] = red
            print(json.dumps(line), flush=True)
        dist.barrier()
        dist.destroy_process_group()
    elif line is not None:
        print(json.dumps(line), flush=True)
    return line


def main():
    a = parse()
    if a.impl == "reference":
        run_reference(a)
    elif a.workload == "dropout":
        run_ours(a)
    else:
        from tools import bench_extra
        bench_extra.run(a)


if __name__ == "__main__":
    main()
