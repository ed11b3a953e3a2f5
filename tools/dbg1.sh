cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out/dbg4
timeout 900 python tools/stress_repro.py --case 25 --case 29 --reps 10 > gpurun_out/dbg4/repro.log 2>&1
timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/dbg4/pytest.log 2>&1
cat gpurun_out/dbg4/repro.log | grep -v "^$" | tail -20; grep "^FAILED" gpurun_out/dbg4/pytest.log; tail -2 gpurun_out/dbg4/pytest.log
