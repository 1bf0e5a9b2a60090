#!/bin/bash
# Evidence for profiles/: bench lines, launch list of the bench command, ncu --set full captures.
# PART=a: bench lines + launch list + dropout capture; PART=b: init / pack / Normal captures.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
shrink() {  # export CSV pages on the box; drop reports too large to copy back
  for r in gpurun_out/*.ncu-rep; do
    ncu -i "$r" --page raw --csv > "${r%.ncu-rep}.raw.csv" 2>/dev/null
    ncu -i "$r" --page source --csv --print-source sass > "${r%.ncu-rep}.src.csv" 2>/dev/null
    [ "$(stat -c %s "$r")" -gt 12000000 ] && rm -f "$r"
  done
}
if [ "$PART" != "b" ]; then
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > gpurun_out/gpu.txt 2>&1
timeout 600 python bench.py > gpurun_out/bench.log 2>&1
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1
rm -f gpurun_out/bench_extra.log
for w in randn embed init redistribute; do timeout 600 python bench.py --workload $w --steps 5 --warmup 3 >> gpurun_out/bench_extra.log 2>&1; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_dropout_fast -s 4 -c 1 -o gpurun_out/prof_dropout -f python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
else
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fill_batch -c 1 -o gpurun_out/prof_init -f python bench.py --workload init --steps 1 --warmup 0 > gpurun_out/ncu_init.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_copy_tiles -c 1 -o gpurun_out/prof_pack -f python tools/time_pack.py > gpurun_out/ncu_pack.log 2>&1
bash tools/gpu_prof_normal.sh
fi
shrink
du -sh gpurun_out
