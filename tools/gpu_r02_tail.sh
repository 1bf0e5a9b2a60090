#!/bin/bash
# Round-2 tail pass after the float64 Normal corrections: smoke, full GPU suite, the randn line
# (with its float64 sub-object) and an ncu capture of the float64 Normal fill.
mkdir -p gpurun_out/r02tail; O=gpurun_out/r02tail
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest.txt 2>&1; echo "pytest rc=$?" >> $O/pytest.txt
timeout 600 python bench.py --workload randn --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_randn.txt 2>&1
SDR_NORMAL_DEBUG=1 timeout 300 python tools/time_fill_dtypes.py > $O/dtypes.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_fill_fast -c 1 -o $O/prof_f64 -f python tools/time_fill_dtypes.py > $O/ncu.log 2>&1
ncu -i $O/prof_f64.ncu-rep --page raw --csv > $O/prof_f64.raw.csv 2>/dev/null; rm -f $O/prof_f64.ncu-rep
tail -1 $O/smoke.txt; tail -2 $O/pytest.txt; grep '^{' $O/bench_randn.txt | cut -c1-400; cat $O/dtypes.txt
