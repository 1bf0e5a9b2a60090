#!/bin/bash
# Round-2 pass B: bench line (parity, probes, cpu info), peer self-check in the
# GPU peer tests, and the N-rank bench with the cfg5 redistribute sub-object.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "peer or redistribute" > gpurun_out/r02b_pytest.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/r02b_pytest.txt
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r02b_bench1.txt 2>&1
./tools/gpu_multirank.sh
tail -2 gpurun_out/r02b_pytest.txt; tail -c 2500 gpurun_out/multirank_4.log
