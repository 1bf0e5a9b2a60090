#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
for rep in 1 2; do for f in variants/*.so; do echo "== $f"; SDR_LIB_PATH=$f timeout 300 python tools/time_kernels.py 2>&1 | head -12; done; done > gpurun_out/ab_walk.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
