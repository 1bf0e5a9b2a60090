#!/bin/bash
# Round-2 pass F (re-entry): full GPU tests, smoke, bench headline + every workload.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r02f_smi.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02f_smoke.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/r02f_pytest.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/r02f_pytest.txt
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r02f_bench.txt 2>&1
for w in randn embed init redistribute peer; do
  timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --workload $w >> gpurun_out/r02f_bench_w.txt 2>&1
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r02f_bench_ref.txt 2>&1
tail -3 gpurun_out/r02f_smoke.txt gpurun_out/r02f_pytest.txt; tail -1 gpurun_out/r02f_bench.txt; grep '^{' gpurun_out/r02f_bench_w.txt | cut -c1-400
