#!/bin/bash
# A/B timing of variants/*.so (2 passes) -> gpurun_out/ab_<tag>.log
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
tag=${1:-x}
for rep in 1 2; do for f in variants/*.so; do SDR_LIB_PATH=$f timeout 180 python tools/time_ab.py; done; done > gpurun_out/ab_$tag.log 2>&1
cat gpurun_out/ab_$tag.log
