cd "${GRAFT_REPO_ROOT:-/root/repo}"; O=gpurun_out/x19; mkdir -p $O
GFS_MOSAIC_EXTRAS='[{}, {"gpu.k1_direct": false}, {"gpu.k1_copy": "ldg"}, {}, {"gpu.k1_direct": false}]' timeout 900 python tools/mosaic_probe.py > $O/mosaic.log 2>&1
grep label $O/mosaic.log | cut -c1-330
