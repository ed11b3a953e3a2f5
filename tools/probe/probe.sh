#!/bin/bash
# Environment probe for the GPU box: cores, memory, disks, PCIe topology, storage + PCIe bandwidth.
set -x
out=gpurun_out/probe; mkdir -p $out
{ nproc; lscpu | head -30; free -g; df -hT /tmp /root /dev/shm $GRAFT_REPO_ROOT; mount | grep -E ' / | /tmp | /root ' ; lsblk -o NAME,SIZE,TYPE,MOUNTPOINT,ROTA,MODEL 2>&1 | head -40;
  cat /proc/mdstat 2>&1; nvidia-smi; nvidia-smi topo -m; nvidia-smi -q | grep -iA6 "PCI$\|Link Width\|GPU Link Info" | head -60; uname -a; cat /proc/sys/kernel/io_uring_disabled; ulimit -a; numactl -H 2>&1 | head; } > $out/env.txt 2>&1
./tools/probe/probe_pcie > $out/pcie.txt 2>&1
for dir in /tmp /dev/shm; do
  f=$dir/gfs_probe.bin
  ./tools/probe/probe_io $f 8192 create >> $out/io_$(basename $dir).txt 2>&1
  timeout 300 ./tools/probe/probe_io $f 8192 >> $out/io_$(basename $dir).txt 2>&1
  rm -f $f
done
