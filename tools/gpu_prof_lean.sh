#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
SDR_LIB_PATH=variants/n2.so timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_fill_fast -s 2 -c 1 -o gpurun_out/prof_n2_f32 -f python tools/prof_normal.py f32 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_fill_fast -s 2 -c 1 -o gpurun_out/prof_lean_bf16 -f python tools/prof_normal.py bf16 > /dev/null 2>&1
for r in gpurun_out/prof_n2_f32 gpurun_out/prof_lean_bf16; do
  ncu -i $r.ncu-rep --page raw --csv > $r.raw.csv 2>/dev/null; ncu -i $r.ncu-rep --page source --csv --print-source sass > $r.src.csv 2>/dev/null; rm -f $r.ncu-rep
done
