#!/bin/bash
# Round-2 pass D: compact Normal mirror (build stats, parity), then A/B of the split variants.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
SDR_NORMAL_DEBUG=1 timeout 900 python -m pytest tests/test_rng_gpu.py tests/test_init_gpu.py tests/test_dropout_gpu.py -m gpu -x -q > gpurun_out/r02d_pytest.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/r02d_pytest.txt
SDR_NORMAL_DEBUG=1 python -c "
import torch, time
from paper_2509_07003_b200 import rng as R
t=time.perf_counter(); R.ensure_normal_tables(); torch.cuda.synchronize(); print('first ensure_normal_tables', time.perf_counter()-t, 's'); print(R.normal_mirror_info())
" > gpurun_out/r02d_mirror.txt 2>&1
./tools/gpu_ab.sh split
tail -3 gpurun_out/r02d_pytest.txt; cat gpurun_out/r02d_mirror.txt
