#!/bin/bash
# float64 Normal per-point corrections: parity tests, dtype timings with and without, ncu of the f64 fill.
set -x
mkdir -p gpurun_out/f64d
export SDR_NORMAL_DEBUG=1
timeout 900 python -m pytest tests/test_rng_gpu.py -x -q -k "float64_normal or fast_paths_equal or mirror or transform_plugin" 2>&1 | tail -15 > gpurun_out/f64d/tests.txt
timeout 300 python tools/time_fill_dtypes.py > gpurun_out/f64d/dtypes_on.txt 2>&1
SDR_NORMAL_F64_DELTA=0 timeout 300 python tools/time_fill_dtypes.py > gpurun_out/f64d/dtypes_off.txt 2>&1
timeout 600 ncu --set full --clock-control none -k regex:k_fill_fast -c 1 --launch-skip 0 -o gpurun_out/f64d/prof_f64 -f python tools/time_fill_dtypes.py > gpurun_out/f64d/ncu.log 2>&1
ncu -i gpurun_out/f64d/prof_f64.ncu-rep --page raw --csv > gpurun_out/f64d/prof_f64.raw.csv 2>/dev/null
cat gpurun_out/f64d/tests.txt gpurun_out/f64d/dtypes_on.txt gpurun_out/f64d/dtypes_off.txt
