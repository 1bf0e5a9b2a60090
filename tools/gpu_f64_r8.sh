#!/bin/bash
# 8-bit r corrections: float64 parity tests, then A/B timing against variants/*.so.
mkdir -p gpurun_out/f64r8
SDR_NORMAL_DEBUG=1 timeout 900 python -m pytest tests/test_rng_gpu.py -x -q -s -k "float64_normal or fast_paths_equal or mirror_is_compact or calibration_and_large" 2>&1 | grep -v "^$" | tail -8 > gpurun_out/f64r8/tests.txt
cat gpurun_out/f64r8/tests.txt
./tools/gpu_ab_f64.sh
