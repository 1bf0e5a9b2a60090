#!/bin/bash
# cfg5 redistribute bench line with N ranks sharing one GPU: peer transport (IPC
# on one device) vs the gloo-staged collectives.  Rates are NOT NVLink rates.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
for t in peer nccl; do for n in 2 4; do
SDR_COMM_CPU_STAGING=1 SDR_TRANSPORT=$t SDR_BENCH_SHARE_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29700+n)) bench.py --workload redistribute --gpus $n --steps 3 --warmup 3 > gpurun_out/mr_peer_${t}_$n.log 2>&1; echo "rc=$?" >> gpurun_out/mr_peer_${t}_$n.log
done; done
