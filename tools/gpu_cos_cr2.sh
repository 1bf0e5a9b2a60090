#!/bin/bash
mkdir -p gpurun_out/coscr; O=gpurun_out/coscr
timeout 900 python -m pytest tests/test_rng_gpu.py -x -q -k "float64_normal or fast_paths_equal or mirror or calibration_and_large or transform_plugin or init" 2>&1 | tail -3 > $O/tests2.txt
cat $O/tests2.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_fill_fast -c 1 -o $O/prof -f python tools/time_fill_dtypes.py > $O/ncu.log 2>&1
ncu -i $O/prof.ncu-rep --page raw --csv > $O/prof.raw.csv 2>/dev/null
ncu -i $O/prof.ncu-rep --page source --csv --print-source sass > $O/prof.src.csv 2>/dev/null; rm -f $O/prof.ncu-rep
