#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_fill_fast -s 2 -c 1 -o gpurun_out/prof_tf_bf16 -f python tools/prof_normal.py bf16 > /dev/null 2>&1
r=gpurun_out/prof_tf_bf16; ncu -i $r.ncu-rep --page raw --csv > $r.raw.csv 2>/dev/null; ncu -i $r.ncu-rep --page source --csv --print-source sass > $r.src.csv 2>/dev/null; rm -f $r.ncu-rep
