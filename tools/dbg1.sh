cd "${GRAFT_REPO_ROOT:-/root/repo}"; O=gpurun_out/x22; mkdir -p $O
C="--cell 64x4K --cell 64x16K --cell 64x64K --cell 128x4K --cell 128x64K --cell 1024x64K"
for ns in 5 4; do
  GFS_TMA_STAGES=$ns timeout 600 python tools/c3_cell.py $C --arm prefetch_static > $O/cells_$ns.log 2>&1
  GFS_TMA_STAGES=$ns timeout 600 python tools/c3_cell.py $C --arm prefetch_adaptive >> $O/cells_$ns.log 2>&1
  for i in 1 2 3; do GFS_TMA_STAGES=$ns timeout 600 python tools/profile_run.py --size-gib 16 >> $O/headline_$ns.log 2>&1; done
  GFS_TMA_STAGES=$ns timeout 600 python tools/consumer_probe.py > $O/cons_$ns.log 2>&1
done
timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider -x > $O/pytest.log 2>&1
for ns in 5 4; do echo "== $ns"; grep -h cell $O/cells_$ns.log | python3 -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['arm'][:16], d['cell'], d['gbps'])"; grep profile_run $O/headline_$ns.log; grep variant $O/cons_$ns.log | cut -c1-60; done
grep "^FAILED" $O/pytest.log | head; tail -2 $O/pytest.log
