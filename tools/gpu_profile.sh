#!/bin/bash
# Evidence for profiles/: bench line, launch list of the bench command, full captures.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/bench.log 2>&1
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1
for w in randn init redistribute; do timeout 600 python bench.py --workload $w --steps 5 --warmup 2 >> gpurun_out/bench_extra.log 2>&1; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_dropout_fast -s 2 -c 1 -o gpurun_out/prof_dropout_r01 -f python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fill_fast -s 3 -c 1 -o gpurun_out/prof_normal_r01 -f python bench.py --workload randn --steps 3 --warmup 2 > gpurun_out/ncu_normal.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fill_batch -c 1 -o gpurun_out/prof_init_r01 -f python bench.py --workload init --steps 1 --warmup 0 > gpurun_out/ncu_init.log 2>&1
