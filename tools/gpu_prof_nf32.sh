cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_fill_fast -s 2 -c 1 -o gpurun_out/prof_nf32b -f python tools/prof_normal.py f32 > gpurun_out/ncu_nf32b.log 2>&1
ncu -i gpurun_out/prof_nf32b.ncu-rep --page raw --csv > gpurun_out/prof_nf32b.raw.csv 2>/dev/null
ncu -i gpurun_out/prof_nf32b.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_nf32b.src.csv 2>/dev/null
rm -f gpurun_out/prof_nf32b.ncu-rep
