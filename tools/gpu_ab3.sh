#!/bin/bash
# A/B timing of variants/*.so (2 passes) + the GPU test suite on the default build.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
for rep in 1 2; do for f in variants/*.so; do SDR_LIB_PATH=$f timeout 180 python tools/time_ab.py; done; done > gpurun_out/ab.log 2>&1
timeout 900 python -m pytest tests -m gpu -q --timeout 800 -x > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
