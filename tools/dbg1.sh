cd "${GRAFT_REPO_ROOT:-/root/repo}"; O=gpurun_out/x3; mkdir -p $O
C="--cell 64x4K --cell 64x16K --cell 64x64K --cell 128x4K --cell 128x64K"
for hp in 1 0; do
timeout 600 python tools/c3_cell.py $C --arm prefetch_static --set gpu.pull_helpers=$hp >> $O/cells.log 2>&1
timeout 600 python tools/c3_cell.py $C --arm prefetch_adaptive --set gpu.pull_helpers=$hp >> $O/cells.log 2>&1
done
timeout 600 python tools/consumer_probe.py > $O/cons_hybrid.log 2>&1
timeout 600 python tools/consumer_probe.py io.transfer=mapped > $O/cons_mapped.log 2>&1
timeout 600 python tools/consumer_probe.py io.transfer=mapped gpu.pull_helpers=0 > $O/cons_mapped_nohelp.log 2>&1
timeout 1800 python -m pytest tests -q -m gpu -p no:cacheprovider -x -k "stress or golden_case or user_kernel or pressure" > $O/pytest.log 2>&1
grep -h cell $O/cells.log | python3 -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['arm'][:16], d['set'], d['cell'], d['gbps'], d['per_cta_ms'])"
for f in $O/cons_*.log; do echo $f; grep variant $f; done; tail -3 $O/pytest.log
