#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
for rep in 1 2; do for f in variants/*.so; do SDR_LIB_PATH=$f timeout 180 python tools/time_pack.py; done; done > gpurun_out/ab_pack.log 2>&1
