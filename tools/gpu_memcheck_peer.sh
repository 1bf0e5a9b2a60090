#!/bin/bash
# compute-sanitizer memcheck over the peer pull kernels (local peers, no barrier).
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_peer_gpu.py -q -x -k local_peers > gpurun_out/peer_local.log 2>&1; echo "rc=$?" >> gpurun_out/peer_local.log
PYTORCH_NO_CUDA_MEMORY_CACHING=1 timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_peer_gpu.py -q -x -k local_peers > gpurun_out/memcheck_peer.txt 2>&1; echo "rc=$?" >> gpurun_out/memcheck_peer.txt
