#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
for rep in 1 2; do for f in variants/*.so; do echo "== $f"; SDR_LIB_PATH=$f timeout 300 python tools/time_kernels.py 2>&1 | grep -i "cfg4"; SDR_LIB_PATH=$f timeout 180 python tools/time_ab.py | cut -c1-300; done; done > gpurun_out/ab_c2l.log 2>&1
timeout 900 python -m pytest tests/test_rng_gpu.py tests/test_init_gpu.py tests/test_acceptance_gpu.py -q -x -k cfg4 > gpurun_out/pytest_c2l.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_c2l.log
