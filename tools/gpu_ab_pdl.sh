#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
for rep in 1 2; do for f in variants/*.so; do echo "== $f"; SDR_LIB_PATH=$f timeout 300 python tools/time_overhead.py 2>&1 | tail -2; done; done > gpurun_out/ab_pdl.log 2>&1
timeout 900 python -m pytest tests/test_dropout_gpu.py -q -x > gpurun_out/pytest_pdl.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_pdl.log
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench_pdl.log 2>&1
