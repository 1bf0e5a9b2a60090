#!/bin/bash
# Round-2 pass C: NormalLut2 path (f32/f16 normals) parity + timing + ncu; MINB A/B variants.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
SDR_NORMAL_DEBUG=1 timeout 900 python -m pytest tests/test_rng_gpu.py tests/test_init_gpu.py -m gpu -x -q > gpurun_out/r02c_pytest.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/r02c_pytest.txt
(SDR_NORMAL_DEBUG=1 timeout 180 python tools/time_ab.py; for f in variants/*.so; do SDR_LIB_PATH=$f timeout 180 python tools/time_ab.py; done) > gpurun_out/r02c_ab.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_fill_fast -s 2 -c 1 -o gpurun_out/prof_nf32_n2 -f python tools/prof_normal.py f32 > gpurun_out/ncu_nf32_n2.log 2>&1
tail -3 gpurun_out/r02c_pytest.txt; cat gpurun_out/r02c_ab.txt
