#!/bin/bash
# Round-2 pass E: r_fast2 seed A/B, redistribute/peer GPU tests (slice kernel), host profile of redistribute_many.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
./tools/gpu_ab.sh seed > /dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -k "redistribute or peer or init or acceptance" > gpurun_out/r02e_pytest.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/r02e_pytest.txt
SDR_PROFILE_HOST=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29533 tools/time_host_redistribute.py > gpurun_out/r02e_host.txt 2>&1
tail -3 gpurun_out/r02e_pytest.txt; sed 's/| calib.*//; s/dropout full.*| normal f32/normal f32/' gpurun_out/ab_seed.log; head -40 gpurun_out/r02e_host.txt
