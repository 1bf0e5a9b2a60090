#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
for f in variants/*.so; do SDR_LIB_PATH=$f timeout 180 python tools/time_ab.py; done > gpurun_out/ab.log 2>&1
timeout 900 python -m pytest tests -m gpu -q --timeout 600 -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python tools/time_kernels.py > gpurun_out/kernels.log 2>&1
