#!/bin/bash
# N-rank bench path on a 1-GPU box (SDR_BENCH_SHARE_GPU=1: all ranks on cuda:0, gloo).
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
for n in 2 4 8; do
SDR_BENCH_SHARE_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29500+n)) bench.py --gpus $n --steps 5 --warmup 3 > gpurun_out/multirank_$n.log 2>&1; echo "rc=$?" >> gpurun_out/multirank_$n.log
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29600 bench.py --impl reference --gpus 2 --steps 2 --warmup 1 > gpurun_out/multirank_ref.log 2>&1; echo "rc=$?" >> gpurun_out/multirank_ref.log
