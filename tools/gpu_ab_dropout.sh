#!/bin/bash
# A/B of variants/*.so on the dropout kernel (time_ab: cfg2 full + P=8 shard), 3 passes,
# with the dropout GPU parity tests run against every variant.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
tag=${1:-x}
for f in "" variants/*.so; do echo "${f:-default}: $(SDR_LIB_PATH=$f timeout 900 python -m pytest tests/test_dropout_gpu.py -m gpu -x -q 2>&1 | tail -1)"; done > gpurun_out/abd_${tag}_pytest.txt
(for rep in 1 2 3; do timeout 180 python tools/time_ab.py; for f in variants/*.so; do SDR_LIB_PATH=$f timeout 180 python tools/time_ab.py; done; done) 2>&1 | sed 's/| normal f32.*//' > gpurun_out/abd_${tag}.txt
cat gpurun_out/abd_${tag}_pytest.txt gpurun_out/abd_${tag}.txt
