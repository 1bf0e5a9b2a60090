#!/bin/bash
# float64 Normal corrections: the whole GPU suite, dtype timings, ncu of the float64 Normal fill.
mkdir -p gpurun_out/f64f
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -5 > gpurun_out/f64f/tests.txt
SDR_NORMAL_DEBUG=1 timeout 300 python tools/time_fill_dtypes.py > gpurun_out/f64f/dtypes.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_fill_fast -c 1 -o gpurun_out/f64f/prof_f64 -f python tools/time_fill_dtypes.py > gpurun_out/f64f/ncu.log 2>&1
ncu -i gpurun_out/f64f/prof_f64.ncu-rep --page raw --csv > gpurun_out/f64f/prof_f64.raw.csv 2>/dev/null
ncu -i gpurun_out/f64f/prof_f64.ncu-rep --page source --csv > gpurun_out/f64f/prof_f64.src.csv 2>/dev/null
cat gpurun_out/f64f/tests.txt gpurun_out/f64f/dtypes.txt
