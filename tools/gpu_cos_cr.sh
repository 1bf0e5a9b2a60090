#!/bin/bash
# c_cr (double-double cosine, correctly rounded outside a flagged band): parity, load statistics, A/B timing.
mkdir -p gpurun_out/coscr; O=gpurun_out/coscr
SDR_NORMAL_DEBUG=1 timeout 900 python -m pytest tests/test_rng_gpu.py -x -q -s -k "float64_normal or fast_paths_equal or mirror_is_compact or calibration_and_large or transform_plugin" 2>&1 | grep -v "^$" | tail -8 > $O/tests.txt
cat $O/tests.txt
# (the band is now the compile-time SDR_COS_TAU; tau 0.02 / 0.05 measured 173.5 / 173.6 us, flagged 4.0% / 10.0%)
for cfg in "SDR_NORMAL_COS_CR=1" "SDR_NORMAL_COS_CR=0"; do
  echo "== $cfg"; env $cfg SDR_NORMAL_DEBUG=1 timeout 300 python tools/time_fill_dtypes.py 2>&1 | grep "corrections\|normal   torch.float64"
done | tee $O/ab.txt
