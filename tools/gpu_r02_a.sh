#!/bin/bash
# Round-2 first GPU pass: microbenchmarks, NCCL shared-GPU probe, GPU tests, quick bench.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r02a_smi.txt
./tools/ubench_fp64 > gpurun_out/r02a_ubench.txt 2>&1
timeout 120 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29511 tools/nccl_share_probe.py > gpurun_out/r02a_nccl_share.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02a_pytest.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/r02a_pytest.txt
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r02a_bench.txt 2>&1
tail -3 gpurun_out/r02a_pytest.txt; cat gpurun_out/r02a_ubench.txt gpurun_out/r02a_nccl_share.txt | tail -20
