#!/bin/bash
# bench lines at the strong-scaling shard sizes emulated on one GPU are not
# possible with torchrun (1 GPU); run N=1 bench + GPU tests.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 900 python -m pytest tests -m gpu -q --timeout 800 -x > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
