#!/bin/bash
# A/B of variants/*.so on the Normal fills (f32 + bf16 [4096,4096]) and the LLaMA-3-8B init, 2 passes,
# plus the Normal GPU parity tests on the default build.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
tag=${1:-x}
SDR_NORMAL_DEBUG=1 timeout 900 python -m pytest tests/test_rng_gpu.py tests/test_init_gpu.py -m gpu -x -q > gpurun_out/ab_${tag}_pytest.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/ab_${tag}_pytest.txt
(for rep in 1 2; do timeout 180 python tools/time_ab.py; for f in variants/*.so; do SDR_LIB_PATH=$f timeout 180 python tools/time_ab.py; done; done) 2>&1 | sed 's/| calib.*//; s/dropout full.*| normal f32/normal f32/' > gpurun_out/ab_${tag}.txt
for f in "" variants/*.so; do echo "${f:-default}: $(SDR_LIB_PATH=$f timeout 300 python bench.py --workload init --steps 3 --warmup 2 --no-cpu-baseline 2>&1 | grep -o '"ms_per_step": [0-9.]*')"; done >> gpurun_out/ab_${tag}.txt
tail -2 gpurun_out/ab_${tag}_pytest.txt; cat gpurun_out/ab_${tag}.txt
