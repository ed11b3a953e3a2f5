cd "${GRAFT_REPO_ROOT:-/root/repo}"; O=gpurun_out/x7; mkdir -p $O
C="--cell 64x4K --cell 64x16K --cell 64x64K --cell 128x64K --cell 1024x64K"
for d in 1 0; do
  for tr in mapped_hybrid mapped; do
    for i in 1 2; do timeout 600 python tools/profile_run.py --size-gib 16 --set io.transfer=$tr --set gpu.k1_direct=$d >> $O/headline.log 2>&1; done
    echo "^ $tr direct=$d" >> $O/headline.log
  done
  timeout 600 python tools/c3_cell.py $C --arm prefetch_static --set gpu.k1_direct=$d >> $O/cells.log 2>&1
  timeout 600 python tools/c3_cell.py $C --arm prefetch_adaptive --set gpu.k1_direct=$d >> $O/cells.log 2>&1
  timeout 600 python tools/consumer_probe.py gpu.k1_direct=$d > $O/cons_d$d.log 2>&1
done
timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider > $O/pytest.log 2>&1
grep -E "profile_run|\^" $O/headline.log
grep -h cell $O/cells.log | python3 -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['arm'][:16], d['set'], d['cell'], d['gbps'], d['per_cta_ms'])"
for f in $O/cons_*.log; do echo $f; grep variant $f; done; grep "^FAILED" $O/pytest.log | head; tail -2 $O/pytest.log
