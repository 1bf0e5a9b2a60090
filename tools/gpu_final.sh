#!/bin/bash
# Round-end confirmation: smoke, full GPU suite, bench (+reference arm), pack capture.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -q --timeout 1200 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1
timeout 600 python tools/time_kernels.py > gpurun_out/kernels.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_copy_tiles -c 1 -o gpurun_out/prof_pack -f python tools/time_pack.py > gpurun_out/ncu_pack.log 2>&1
ncu -i gpurun_out/prof_pack.ncu-rep --page raw --csv > gpurun_out/prof_pack.raw.csv 2>/dev/null; rm -f gpurun_out/prof_pack.ncu-rep
