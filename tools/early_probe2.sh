cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/early2; mkdir -p $O
C="--cell 64x4K --cell 64x16K --cell 64x64K --cell 128x4K --cell 128x64K"
for x in mapped_hybrid mapped; do for e in true false; do
  timeout 600 python tools/c3_cell.py --arm prefetch_static $C --set io.transfer=$x --set gpu.k1_early=$e >> $O/cells.jsonl 2>> $O/cells.err
done; done
GFS_POLL_NS=1000 timeout 600 python tools/c3_cell.py --arm prefetch_static $C --set io.transfer=mapped --set gpu.k1_early=true | sed 's/"set"/"poll":1000,"set"/' >> $O/cells.jsonl 2>> $O/cells.err
python - <<'P'
import json
for l in open("gpurun_out/early2/cells.jsonl"):
    d=json.loads(l); print(d["cell"], d.get("poll",""), d["set"], d["transfer"], d["gbps"], d["per_cta_ms"])
P
tail -3 $O/cells.err
