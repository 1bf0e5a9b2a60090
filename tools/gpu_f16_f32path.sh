#!/bin/bash
# float16 Normal on the table-free float32 path (SDR_NORMAL_F16_F32): GPU rng/init/dropout tests and dtype timings.
mkdir -p gpurun_out/f16; O=gpurun_out/f16
timeout 1200 python -m pytest tests/test_rng_gpu.py tests/test_init_gpu.py -x -q 2>&1 | tail -3 > $O/tests.txt
cat $O/tests.txt
timeout 300 python tools/time_fill_dtypes.py 2>&1 | grep "normal" | tee $O/dtypes.txt
