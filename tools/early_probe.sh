#!/bin/bash
# K1 early A/B on the C3 static cells, then the GPU test suite.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/${1:-early}; mkdir -p $O
for e in true false true; do
  timeout 600 python tools/c3_cell.py --arm prefetch_static --cell 64x4K --cell 64x16K --cell 64x64K \
    --cell 128x4K --cell 256x64K --cell 1024x64K --set gpu.k1_early=$e >> $O/cells.jsonl 2>> $O/cells.err
done
if [ "$2" != "no-tests" ]; then
  timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider --maxfail=10 > $O/pytest_gpu.log 2>&1
  echo "pytest rc=$?" >> $O/pytest_gpu.log
fi
cat $O/cells.jsonl | cut -c1-200; tail -3 $O/cells.err; tail -3 $O/pytest_gpu.log
