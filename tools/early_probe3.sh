#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/early3; mkdir -p $O
C="--cell 64x4K --cell 64x16K --cell 64x64K --cell 128x4K --cell 256x64K"
for i in 1 2; do for e in true false; do
  timeout 600 python tools/c3_cell.py --arm prefetch_static $C --set gpu.k1_early=$e >> $O/cells.jsonl 2>> $O/cells.err
done; done
python - <<'P'
import json
for l in open("gpurun_out/early3/cells.jsonl"):
    d=json.loads(l); print(d["cell"], d["set"], d["gbps"], d["early_answers"], d["rpc_count"], d["per_cta_ms"])
P
tail -3 $O/cells.err
timeout 1200 python -m pytest tests -q -m gpu -p no:cacheprovider -x -k "mapped or stress or user_kernel or smoke" > $O/pytest.log 2>&1; tail -3 $O/pytest.log
