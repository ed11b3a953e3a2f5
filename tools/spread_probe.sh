#!/bin/bash
# first-wave TB placement (one TB per SM) A/B on C3 / C4 shapes with few TBs
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/${1:-spread}; mkdir -p $O
C="--cell 64x4K --cell 64x16K --cell 64x64K --cell 128x4K --cell 128x64K --cell 256x4K"
for i in 1 2; do for sp in 1 0; do for e in true false; do
  GFS_SPREAD=$sp timeout 600 python tools/c3_cell.py --arm prefetch_static $C --timeline --set gpu.k1_early=$e | sed "s/\"set\"/\"spread\":$sp,\"set\"/" >> $O/cells.jsonl 2>> $O/cells.err
done; done; done
for sp in 1 0; do
  GFS_SPREAD=$sp timeout 600 python tools/c3_cell.py --arm prefetch_adaptive $C | sed "s/\"set\"/\"spread\":$sp,\"set\"/" >> $O/cells.jsonl 2>> $O/cells.err
done
python - <<'P'
import json
for l in open("gpurun_out/spread/cells.jsonl"):
    d=json.loads(l); print(d["cell"], d["arm"][9:], d.get("spread"), d["set"], d["gbps"], d.get("tb_end_ms_p10_p50_max"))
P
tail -3 $O/cells.err
