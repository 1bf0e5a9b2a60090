#!/bin/bash
# Round-2 pass H: A/B of warp-specialised Normal variants (variants/*.so), 2 passes.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
(for rep in 1 2; do timeout 180 python tools/time_ab.py; for f in variants/*.so; do SDR_LIB_PATH=$f timeout 180 python tools/time_ab.py; done; done) 2>&1 | sed 's/| calib.*//; s/dropout full.*| normal f32/normal f32/' > gpurun_out/r02h_ab.txt
cat gpurun_out/r02h_ab.txt
