cd "${GRAFT_REPO_ROOT:-/root/repo}"; O=gpurun_out/x14; mkdir -p $O
C="--cell 64x4K --cell 64x16K --cell 64x64K --cell 128x4K --cell 128x64K --cell 1024x64K"
timeout 600 python tools/c3_cell.py $C --arm prefetch_static >> $O/cells.log 2>&1
timeout 600 python tools/c3_cell.py $C --arm prefetch_adaptive >> $O/cells.log 2>&1
for i in 1 2 3; do timeout 600 python tools/profile_run.py --size-gib 16 >> $O/headline.log 2>&1; done
for i in 1 2; do timeout 600 python tools/profile_run.py --size-gib 16 --set io.transfer=bounce >> $O/headline.log 2>&1; done
timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider -x > $O/pytest.log 2>&1
grep -h cell $O/cells.log | python3 -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['arm'][:16], d['cell'], d['gbps'], d['kernel_ms'], d['per_cta_ms'])"
grep profile_run $O/headline.log; grep "^FAILED" $O/pytest.log | head; tail -2 $O/pytest.log
