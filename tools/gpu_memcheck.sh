#!/bin/bash
# compute-sanitizer memcheck / racecheck over the smoke test and the small GPU tests.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
export PYTORCH_NO_CUDA_MEMORY_CACHING=1
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/memcheck_smoke.txt 2>&1
timeout 1500 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_init_gpu.py tests/test_dropout_gpu.py -q -x -k "not large and not 64bit and not cfg4 and not cfg2" > gpurun_out/memcheck_tests.txt 2>&1
timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/racecheck_smoke.txt 2>&1
timeout 900 compute-sanitizer --tool synccheck --print-limit 20 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/synccheck_smoke.txt 2>&1
timeout 1200 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_rng_gpu.py -q -x -k "sharded_fill and 65536" > gpurun_out/memcheck_fill.txt 2>&1
