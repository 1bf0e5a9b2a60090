#!/bin/bash
# ncu --set full (with source) of the warp-specialised Normal fill: f32 and bf16 [4096,4096].
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
for w in ${WS_WHICH:-f32 bf16}; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:${WS_KERNEL:-k_fill_normal_ws} -s 2 -c 1 -o gpurun_out/prof_ws_$w -f python tools/prof_normal.py $w > gpurun_out/ncu_ws_$w.log 2>&1
  ncu -i gpurun_out/prof_ws_$w.ncu-rep --page raw --csv > gpurun_out/prof_ws_$w.raw.csv 2>/dev/null
  ncu -i gpurun_out/prof_ws_$w.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_ws_$w.src.csv 2>/dev/null
  rm -f gpurun_out/prof_ws_$w.ncu-rep
done
ls -la gpurun_out/
