cd "${GRAFT_REPO_ROOT:-/root/repo}"; O=gpurun_out/x16; mkdir -p $O
timeout 600 python tools/preset_probe.py > $O/preset.log 2>&1
timeout 600 python tools/preset_probe.py --set gpu.k1_direct=0 > $O/preset_nodirect.log 2>&1
GFS_CE_MIN_KIB=1000000 timeout 600 python tools/preset_probe.py --set io.transfer=mapped_hybrid > $O/preset_doorbell.log 2>&1
for f in $O/preset*.log; do echo $f; cat $f | grep arm; done
