"""Host (Python) time per redistribute_many call on the peer transport: the
cfg5 layer, AG over dp=2, ranks sharing one GPU (gloo for the one-time heap
exchange).  torchrun --nproc-per-node 2 tools/time_host_redistribute.py"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.distributed as dist
torch.cuda.set_device(0)
dist.init_process_group("gloo")
from paper_2509_07003_b200 import create_mesh
from paper_2509_07003_b200.dtensor import from_local, redistribute_many
from paper_2509_07003_b200.placement import ShardSpec, local_shape_and_offset, parse_placements
rank = dist.get_rank()
mesh = create_mesh([("dp", 2)])
coord = mesh.coords_of_rank(rank)
d, ff, kv = 4096, 14336, 1024
layer = {"q": ((d, d), "S(1)"), "k": ((kv, d), "S(1)"), "v": ((kv, d), "S(1)"), "o": ((d, d), "S(0)"),
         "gate": ((ff, d), "S(1)"), "up": ((ff, d), "S(1)"), "down": ((d, ff), "S(0)"), "n1": ((d,), "S(0)"),
         "n2": ((d,), "S(0)")}
xs, dsts = [], []
for shape, pl in layer.values():
    spec = ShardSpec(mesh, parse_placements(pl))
    v = local_shape_and_offset(spec, shape, coord)
    xs.append(from_local(torch.randn(v.local_shape, device="cuda", dtype=torch.bfloat16), spec, shape, coord))
    dsts.append(ShardSpec(mesh, parse_placements("R")))
for _ in range(3):
    redistribute_many(xs, dsts)
torch.cuda.synchronize()
dist.barrier()
ts = []
for _ in range(20):
    t0 = time.perf_counter()
    ys = redistribute_many(xs, dsts)
    ts.append(time.perf_counter() - t0)
    torch.cuda.synchronize()
    dist.barrier()
ts.sort()
# breakdown: the peer C call (pack + barrier + pull launches) and the output allocation
from paper_2509_07003_b200 import peer as _peer, dtensor as _dt
acc = {"c_call": 0.0, "alloc": 0.0, "n": 0}
_ag, _al = _peer.PeerHeap.all_gather_arrays, _dt._alloc_outputs
def _ag_t(self, *a, **k):
    t = time.perf_counter(); r = _ag(self, *a, **k); acc["c_call"] += time.perf_counter() - t; return r
def _al_t(*a, **k):
    t = time.perf_counter(); r = _al(*a, **k); acc["alloc"] += time.perf_counter() - t; return r
_peer.PeerHeap.all_gather_arrays, _dt._alloc_outputs = _ag_t, _al_t
t_all = 0.0
for _ in range(20):
    t0 = time.perf_counter()
    redistribute_many(xs, dsts)
    t_all += time.perf_counter() - t0
    acc["n"] += 1
    torch.cuda.synchronize()
    dist.barrier()
_peer.PeerHeap.all_gather_arrays, _dt._alloc_outputs = _ag, _al
if rank == 0:
    n = acc["n"]
    print(f"breakdown per call: total {t_all/n*1e6:.0f} us = peer C call(s) {acc['c_call']/n*1e6:.0f} us "
          f"+ output allocation {acc['alloc']/n*1e6:.0f} us + the rest (plan lookup, pointer patching) "
          f"{(t_all-acc['c_call']-acc['alloc'])/n*1e6:.0f} us", flush=True)
if rank == 0:
    print(f"host time per redistribute_many (9 members, peer): median {ts[len(ts)//2]*1e6:.0f} us, "
          f"min {ts[0]*1e6:.0f} us", flush=True)
if os.environ.get("SDR_PROFILE_HOST") == "1":
    import cProfile, pstats
    pr = cProfile.Profile()
    pr.enable()
    for _ in range(200):
        redistribute_many(xs, dsts)
    pr.disable()
    torch.cuda.synchronize()
    if rank == 0:
        pstats.Stats(pr).sort_stats("tottime").print_stats(25)
dist.barrier()
dist.destroy_process_group()
