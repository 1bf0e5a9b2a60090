cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
for w in randn embed init redistribute; do
SDR_BENCH_SHARE_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29561 bench.py --workload $w --gpus 4 --steps 3 --warmup 2 >> gpurun_out/bench_mr.log 2>&1; echo "$w rc=$?" >> gpurun_out/bench_mr.log
done
