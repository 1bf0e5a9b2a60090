#!/bin/bash
# float16 Normal: MUFU cosine (main) vs the table cosine (variants/f16tab.so), parity + timing.
mkdir -p gpurun_out/f16; O=gpurun_out/f16
SDR_LIB_PATH=variants/f16tab.so timeout 900 python -m pytest tests/test_rng_gpu.py -x -q -k "float16 or fast_paths or golden or oracle" 2>&1 | tail -1
for pass in 1 2; do for v in main variants/f16tab.so; do
  if [ "$v" = main ]; then unset SDR_LIB_PATH; else export SDR_LIB_PATH=$v; fi
  echo "== $v"; timeout 300 python tools/time_fill_dtypes.py 2>&1 | grep "normal   torch.float16\|normal   torch.bfloat16"
done; done | tee $O/ab.txt
