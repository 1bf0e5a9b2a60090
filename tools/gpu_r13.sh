#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 800 -x > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python tools/time_kernels.py > gpurun_out/kernels.log 2>&1
timeout 300 python bench.py --workload init --steps 3 --warmup 1 > gpurun_out/bench_init.log 2>&1
