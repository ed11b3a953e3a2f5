cd "${GRAFT_REPO_ROOT:-/root/repo}"; O=gpurun_out/x17; mkdir -p $O
C="--cell 64x4K --cell 64x64K --cell 128x4K --cell 128x64K --cell 1024x64K"
for p in 4000 1000 500 250; do
  GFS_POLL_NS=$p timeout 600 python tools/c3_cell.py $C --arm prefetch_static > $O/cells_$p.log 2>&1
  GFS_POLL_NS=$p timeout 600 python tools/consumer_probe.py > $O/cons_$p.log 2>&1
  GFS_POLL_NS=$p timeout 600 python tools/preset_probe.py > $O/preset_$p.log 2>&1
done
for p in 4000 1000 500 250; do echo "== $p"; grep -h cell $O/cells_$p.log | python3 -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['cell'], d['gbps'], d['per_cta_ms']['wait_ns'])"; grep variant $O/cons_$p.log | cut -c1-60; grep '"rep": 2' $O/preset_$p.log | cut -c1-80; done
