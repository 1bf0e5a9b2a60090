#!/bin/bash
# Round-2 pass I: MUFU bfloat16 Normal -- calibration, parity (rng + init GPU tests), A/B vs table path, init bench.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
SDR_NORMAL_DEBUG=1 timeout 900 python -m pytest tests/test_rng_gpu.py tests/test_init_gpu.py -m gpu -x -q > gpurun_out/r02i_pytest.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/r02i_pytest.txt
(for rep in 1 2; do timeout 180 python tools/time_ab.py; for f in variants/*.so; do SDR_LIB_PATH=$f timeout 180 python tools/time_ab.py; done; done) 2>&1 | sed 's/| calib.*//; s/dropout full.*| normal f32/normal f32/' > gpurun_out/r02i_ab.txt
for f in "" variants/nomufu.so variants/mufu3.so; do SDR_LIB_PATH=$f timeout 300 python bench.py --workload init --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | grep '^{' | cut -c1-330; done > gpurun_out/r02i_init.txt
grep -h "sdr normal mirror" gpurun_out/r02i_pytest.txt | head -2; tail -3 gpurun_out/r02i_pytest.txt; cat gpurun_out/r02i_ab.txt gpurun_out/r02i_init.txt
