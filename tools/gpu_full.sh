#!/bin/bash
# Round-end style pass on one box: all GPU tests, smoke, bench of record, reference arm,
# ncu launch list of the bench command and one --set full capture of gread_driver.
# usage: tools/gpu_full.sh <tag> [skip-tests]
cd "${GRAFT_REPO_ROOT:-/root/repo}"
T=${1:-run}; O=gpurun_out/$T; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt 2>&1
nvidia-smi topo -m > $O/topo.txt 2>&1
if [ "$2" != "skip-tests" ]; then
  timeout 2700 python -m pytest tests -q -m gpu -p no:cacheprovider --maxfail=10 > $O/pytest_gpu.log 2>&1
  echo "pytest rc=$?" >> $O/pytest_gpu.log
fi
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 1200 python bench.py > $O/bench.log 2>&1; echo "bench rc=$?" >> $O/bench.log
timeout 900 python bench.py --impl reference > $O/bench_ref.log 2>&1; echo "ref rc=$?" >> $O/bench_ref.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv \
  python bench.py --quick --steps 2 --warmup 1 --no-clocks > $O/bench_ncu.log 2>&1
timeout 1200 ncu --replay-mode application --set full --clock-control none --import-source on -k regex:gread_driver -c 1 -o $O/gread_full -f \
  python tools/profile_run.py --size-gib 2 > $O/ncu_full.log 2>&1
tail -3 $O/pytest_gpu.log 2>/dev/null; tail -2 $O/smoke.log; tail -c 1200 $O/bench.log; tail -c 600 $O/bench_ref.log
