#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 600 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench.log 2>&1
timeout 600 python tools/time_kernels.py > gpurun_out/kernels.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fill_fast -s 3 -c 1 -o gpurun_out/prof_normal_r01b -f python bench.py --workload randn --steps 3 --warmup 2 > gpurun_out/ncu_normal.log 2>&1
