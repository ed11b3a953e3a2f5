cd "${GRAFT_REPO_ROOT:-/root/repo}"; O=gpurun_out/x6; mkdir -p $O
C="--cell 64x4K --cell 64x16K --cell 64x64K --cell 128x64K"
for hp in 0 1; do
timeout 600 python tools/c3_cell.py $C --arm prefetch_static --set gpu.pull_helpers=$hp >> $O/cells.log 2>&1
timeout 600 python tools/c3_cell.py $C --arm prefetch_adaptive --set gpu.pull_helpers=$hp >> $O/cells.log 2>&1
timeout 600 python tools/consumer_probe.py gpu.pull_helpers=$hp > $O/cons_h$hp.log 2>&1
done
timeout 1500 python tools/sweep_c3.py --out $O/c3.json > $O/c3.log 2>&1
grep -h cell $O/cells.log | python3 -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['arm'][:16], d['set'], d['cell'], d['gbps'], d['per_cta_ms'], d['pull_jobs'], d['helper_chunks'], d['pull_wait_ms_per_cta'])"
for f in $O/cons_*.log; do echo $f; grep variant $f; done; grep "64 4096\|64 16384" $O/c3.log
