#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 800 > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 1200 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_rng_gpu.py tests/test_dropout_gpu.py tests/test_init_gpu.py -q -x -k "golden or empty or sharded_fill_matches_oracle and 65536 or dropout_matches_oracle or materialize or pack" > gpurun_out/memcheck.log 2>&1; echo "rc=$?" >> gpurun_out/memcheck.log
timeout 600 python tools/time_kernels.py > gpurun_out/kernels.log 2>&1
