#!/bin/bash
# ncu --set full captures (with source) of the Normal fill kernels.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_fill_fast -s 2 -c 1 -o gpurun_out/prof_nf32 -f python tools/prof_normal.py f32 > gpurun_out/ncu_nf32.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_fill_fast -s 2 -c 1 -o gpurun_out/prof_nbf16 -f python tools/prof_normal.py bf16 > gpurun_out/ncu_nbf16.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_fill_fast -s 2 -c 1 -o gpurun_out/prof_u32 -f python tools/prof_normal.py u32 > gpurun_out/ncu_u32.log 2>&1
