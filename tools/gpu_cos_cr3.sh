#!/bin/bash
mkdir -p gpurun_out/coscr; O=gpurun_out/coscr
timeout 900 python -m pytest tests/test_rng_gpu.py tests/test_init_gpu.py -x -q -k "float64 or fast_paths_equal or mirror or calibration_and_large or transform_plugin or init or golden" 2>&1 | tail -3 > $O/tests3.txt
cat $O/tests3.txt
for cfg in "SDR_NORMAL_COS_CR=1" "SDR_NORMAL_COS_CR=0"; do
  echo "== $cfg"; env $cfg timeout 300 python tools/time_fill_dtypes.py 2>&1 | grep "normal   torch.float64"
done | tee $O/ab3.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_fill_fast -c 1 -o $O/prof3 -f python tools/time_fill_dtypes.py > $O/ncu3.log 2>&1
ncu -i $O/prof3.ncu-rep --page raw --csv > $O/prof3.raw.csv 2>/dev/null; rm -f $O/prof3.ncu-rep
