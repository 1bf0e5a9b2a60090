#!/bin/bash
# All bench lines for profiles/r01_bench.jsonl.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
rm -f gpurun_out/benchlines.jsonl
timeout 600 python bench.py > gpurun_out/b_main.log 2>&1
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/b_ref.log 2>&1
for w in randn embed init redistribute peer; do timeout 600 python bench.py --workload $w --steps 5 --warmup 3 > gpurun_out/b_$w.log 2>&1; done
grep -h '^{' gpurun_out/b_main.log gpurun_out/b_ref.log gpurun_out/b_randn.log gpurun_out/b_embed.log gpurun_out/b_init.log gpurun_out/b_redistribute.log gpurun_out/b_peer.log > gpurun_out/benchlines.jsonl
