"""Can two NCCL ranks share one GPU on this box?  (Decides whether the NCCL
leg of redistribute can be exercised by a 1-GPU test.)
    torchrun --nproc-per-node 2 --master-addr 127.0.0.1 tools/nccl_share_probe.py"""
import os
import torch
import torch.distributed as dist

rank = int(os.environ["RANK"])
torch.cuda.set_device(0)
try:
    dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
    t = torch.full((4,), float(rank + 1), device="cuda")
    dist.all_reduce(t)
    torch.cuda.synchronize()
    print(f"rank {rank}: nccl all_reduce on a shared GPU ok -> {t.tolist()}", flush=True)
    dist.destroy_process_group()
except Exception as e:  # noqa: BLE001
    print(f"rank {rank}: nccl on a shared GPU FAILED: {type(e).__name__}: {str(e)[:300]}", flush=True)
