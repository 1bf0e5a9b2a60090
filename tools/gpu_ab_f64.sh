#!/bin/bash
# A/B of the float64 Normal correction variants (variants/*.so) on [4096,4096] fills.
mkdir -p gpurun_out/f64ab
for pass in 1 2; do
  for v in main variants/*.so; do
    if [ "$v" = main ]; then unset SDR_LIB_PATH; else export SDR_LIB_PATH=$v; fi
    echo "== $v pass $pass"; timeout 300 python tools/time_fill_dtypes.py 2>&1 | grep "normal   torch.float64\|normal   torch.float32"
  done
done 2>&1 | tee gpurun_out/f64ab/ab.txt
