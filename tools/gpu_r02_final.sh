#!/bin/bash
# Round-2 evidence pass: smoke, full GPU tests, bench lines (headline + every workload + reference arm),
# the N-rank bench on one GPU, the ncu launch list of the bench command and ncu --set full captures
# of the headline dropout kernel and the LLaMA-3-8B init kernel (CSV pages exported on the box).
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out/r02final; O=gpurun_out/r02final
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > $O/gpu.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q > $O/pytest.txt 2>&1; echo "pytest rc=$?" >> $O/pytest.txt
timeout 600 python bench.py > $O/bench.txt 2>&1
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.txt 2>&1
for w in randn embed init redistribute peer; do timeout 600 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline >> $O/bench_w.txt 2>&1; done
SDR_BENCH_SHARE_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29502 bench.py --gpus 2 --steps 5 --warmup 3 > $O/multirank_2.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file $O/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $O/ncu_launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_dropout_fast -s 4 -c 1 -o $O/prof_dropout -f python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $O/ncu_dropout.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fill_batch -c 1 -o $O/prof_init -f python bench.py --workload init --steps 1 --warmup 0 --no-cpu-baseline > $O/ncu_init.log 2>&1
for r in $O/*.ncu-rep; do
  ncu -i "$r" --page raw --csv > "${r%.ncu-rep}.raw.csv" 2>/dev/null
  ncu -i "$r" --page source --csv --print-source sass > "${r%.ncu-rep}.src.csv" 2>/dev/null
  rm -f "$r"
done
tail -2 $O/smoke.txt $O/pytest.txt; tail -1 $O/bench.txt | cut -c1-300; du -sh $O
