#!/bin/bash
# Sweep of the host-side data path (see probe_daemon.cu); file on tmpfs, 8 GiB.
set -e
out=gpurun_out/probe; mkdir -p $out
f=/dev/shm/gfs_probe_daemon.bin
[ -f $f ] || ./tools/probe/probe_io $f 8192 create > /dev/null
P=./tools/probe/probe_daemon
{
for mode in zc dma; do
  for T in 8 12 16; do
    for span in 64 2048; do
      for pool in 32 1200; do
        timeout 60 $P $f 8192 $T $span $pool $mode 1
      done
    done
  done
done
timeout 60 $P $f 8192 12 2048 32 dma 0
timeout 60 $P $f 8192 16 4096 64 dma 1
timeout 60 $P $f 8192 16 1024 32 dma 1
} > $out/daemon.txt 2>&1
rm -f $f
