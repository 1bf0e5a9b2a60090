#!/bin/bash
mkdir -p gpurun_out/coscr; O=gpurun_out/coscr
timeout 900 python -m pytest tests/test_rng_gpu.py tests/test_init_gpu.py -x -q -k "float64 or fast_paths_equal or mirror or calibration_and_large or transform_plugin or init or golden" 2>&1 | tail -2 > $O/tests4.txt
cat $O/tests4.txt
for pass in 1 2; do
for v in main variants/nocarve.so; do
  if [ "$v" = main ]; then unset SDR_LIB_PATH; else export SDR_LIB_PATH=$v; fi
  for cfg in "SDR_NORMAL_COS_CR=1" "SDR_NORMAL_COS_CR=0"; do
    echo "== $v $cfg"; env $cfg timeout 300 python tools/time_fill_dtypes.py 2>&1 | grep "normal   torch.float64"
  done
done; done | tee $O/ab4.txt
unset SDR_LIB_PATH
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_fill_fast -c 1 -o $O/prof4 -f python tools/time_fill_dtypes.py > $O/ncu4.log 2>&1
ncu -i $O/prof4.ncu-rep --page raw --csv > $O/prof4.raw.csv 2>/dev/null; rm -f $O/prof4.ncu-rep
