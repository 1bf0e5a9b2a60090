#!/bin/bash
# float64 Normal after the NormalMirror slimming: parity subset, dtype timings, init bench x3.
mkdir -p gpurun_out/f64t; O=gpurun_out/f64t
timeout 900 python -m pytest tests/test_rng_gpu.py tests/test_init_gpu.py -x -q -k "float64 or fast_paths_equal or mirror or calibration_and_large or transform_plugin or init or golden" 2>&1 | tail -2 > $O/tests.txt
cat $O/tests.txt
SDR_NORMAL_DEBUG=1 timeout 300 python tools/time_fill_dtypes.py 2>&1 | grep "corrections\|normal" | tee $O/dtypes.txt
for i in 1 2 3; do timeout 600 python bench.py --workload init --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('init', d['ms_per_step'], d['roofline']['frac'])"; done | tee $O/init.txt
