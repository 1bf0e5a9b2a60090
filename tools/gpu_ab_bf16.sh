#!/bin/bash
# A/B of variants/*.so on the bfloat16 Normal fill and the LLaMA-3-8B init (3 init samples each), with the
# bfloat16 fast-vs-exact parity tests against every variant.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
tag=${1:-x}
for f in "" variants/*.so; do echo "${f:-default}: $(SDR_LIB_PATH=$f timeout 600 python -m pytest tests/test_rng_gpu.py tests/test_init_gpu.py -m gpu -q -x -k 'fast_paths or cfg4 or bfloat16' 2>&1 | tail -1)"; done > gpurun_out/abb_${tag}_pytest.txt
(for rep in 1 2; do for f in "" variants/*.so; do SDR_LIB_PATH=$f timeout 180 python tools/time_ab.py 2>&1 | sed 's/| calib.*//; s/dropout full.*| normal f32/normal f32/' | sed "s|^default|${f:-default}|"; done; done) > gpurun_out/abb_${tag}.txt 2>&1
for f in "" variants/*.so; do echo "${f:-default} init: $(for i in 1 2 3; do SDR_LIB_PATH=$f python bench.py --workload init --steps 3 --warmup 2 --no-cpu-baseline 2>&1 | grep -o '"ms_per_step": [0-9.]*' | cut -d' ' -f2; done | tr '\n' ' ')"; done >> gpurun_out/abb_${tag}.txt
SDR_NORMAL_DEBUG=1 SDR_LIB_PATH=variants/tf256.so python -c "from paper_2509_07003_b200 import rng as R; R.ensure_normal_tables()" 2>&1 | grep calibration >> gpurun_out/abb_${tag}.txt
cat gpurun_out/abb_${tag}_pytest.txt gpurun_out/abb_${tag}.txt
