#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over the round-2 kernels (tools/sanitize_r02.py).
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out; O=gpurun_out/r02_sanitize.txt; : > $O
export PYTORCH_NO_CUDA_MEMORY_CACHING=1
for tool in memcheck racecheck synccheck; do
  for path in "" f64; do
    echo "== $tool SDR_NORMAL_PATH=${path:-default}" >> $O
    SDR_NORMAL_PATH=$path timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_r02.py 2>&1 | grep -E "ok|SUMMARY|Error|error|hazard" | head -12 >> $O
  done
done
echo "== memcheck smoke" >> $O
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | grep -E "ok|SUMMARY" >> $O
cat $O
