#!/bin/bash
# Round-2 pass G: warp-specialised Normal fill -- parity (rng GPU tests) and A/B of producer/consumer splits.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
SDR_NORMAL_DEBUG=1 timeout 900 python -m pytest tests/test_rng_gpu.py -m gpu -x -q > gpurun_out/r02g_pytest.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/r02g_pytest.txt
(for rep in 1 2; do timeout 180 python tools/time_ab.py; for f in variants/*.so; do SDR_LIB_PATH=$f timeout 180 python tools/time_ab.py; done; done) 2>&1 | sed 's/| calib.*//' > gpurun_out/r02g_ab.txt
tail -3 gpurun_out/r02g_pytest.txt; cat gpurun_out/r02g_ab.txt
