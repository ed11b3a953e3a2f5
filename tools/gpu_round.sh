#!/bin/bash
# One GPU-box pass: build check, selected GPU tests, smoke, a quick bench line.
# usage: tools/gpu_round.sh "<pytest -k expr or empty>" [bench args...]
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
K="$1"; shift
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
if [ -n "$K" ]; then
  timeout 2400 python -m pytest tests --maxfail=6 -q -m gpu -k "$K" -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
  echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
fi
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
if [ "$#" -gt 0 ]; then
  timeout 1200 python bench.py "$@" > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
fi
tail -5 gpurun_out/pytest_gpu.log 2>/dev/null; tail -2 gpurun_out/smoke.log; tail -c 1500 gpurun_out/bench.log 2>/dev/null
