#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for rep in 1 2; do python tools/time_ab.py 2>&1 | sed 's/| calib.*//; s/dropout full.*| normal f32/normal f32/'; SDR_LIB_PATH=variants/skipmiss.so python tools/time_ab.py 2>&1 | sed 's/| calib.*//; s/dropout full.*| normal f32/normal f32/'; done
for f in "" variants/skipmiss.so; do echo "${f:-default} init: $(SDR_LIB_PATH=$f python bench.py --workload init --steps 3 --warmup 2 --no-cpu-baseline 2>&1 | grep -o '"ms_per_step": [0-9.]*')"; done
